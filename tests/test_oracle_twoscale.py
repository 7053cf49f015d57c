"""Pins of the oracle's two-scale coarse path (SPEC:364-391 examples, conservation,
the N_B = 1 identity and a coarse cantilever against a direct solve on its own grid)."""
import numpy as np
import pytest

from oracle import fem, grid, sens, solve, twoscale


def test_coarsen_spec_examples():
    # uniform -> uniform; N_B = 1 -> identity; 2x2x2 alternating -> 0.5
    z = np.full(4 * 6 * 2, 0.37)
    assert np.allclose(twoscale.coarsen(z, 4, 6, 2, 2), 0.37, rtol=0, atol=0)
    r = np.random.default_rng(0).uniform(0, 1, 5 * 3 * 7)
    assert np.array_equal(twoscale.coarsen(r, 5, 3, 7, 1), r)
    alt = np.array([0, 1, 0, 1, 0, 1, 0, 1], dtype=float)
    assert np.array_equal(twoscale.coarsen(alt, 2, 2, 2, 2), [0.5])


def test_coarsen_block_bruteforce():
    nx, ny, nz, nb = 6, 4, 8, 2
    z = np.random.default_rng(1).uniform(0, 1, nx * ny * nz)
    zc = twoscale.coarsen(z, nx, ny, nz, nb)
    cx, cy = nx // nb, ny // nb
    for K in range(nz // nb):
        for J in range(cy):
            for I in range(cx):
                s = [z[i + nx * (j + ny * k)] for k in range(K * nb, K * nb + nb)
                     for j in range(J * nb, J * nb + nb) for i in range(I * nb, I * nb + nb)]
                assert abs(zc[I + cx * (J + cy * K)] - np.mean(s)) <= 1e-15
    # volume (sum) is preserved up to the factor nb^3
    assert abs(zc.sum() * nb ** 3 - z.sum()) <= 1e-12 * z.sum()


def test_coarsen_rejects_nondivisible():
    with pytest.raises(ValueError):
        twoscale.coarsen(np.zeros(5 * 4 * 4), 5, 4, 4, 2)


@pytest.mark.parametrize("nb", [1, 2, 4])
def test_restrict_bc_cantilever(nb):
    nx, ny, nz = 8, 4, 4
    fixed, ld, lv = grid.cantilever_bc(nx, ny, nz)
    fc, ldc, lvc = twoscale.restrict_bc(nx, ny, nz, nb, fixed, ld, lv)
    cx, cy, cz = nx // nb, ny // nb, nz // nb
    fcp, _, _ = grid.cantilever_bc(cx, cy, cz)
    assert np.array_equal(fc, fcp)                     # entire coarse face x = 0 fixed
    assert abs(lvc.sum() - lv.sum()) <= 1e-15          # conservation
    assert not fc[ldc].any()
    if nb == 1:                                         # identity
        assert np.array_equal(ldc, ld) and np.array_equal(lvc, lv)


def test_restrict_bc_nearest_rule():
    # ties go up (reading R4): fine index 1 with nb = 2 maps to coarse 1, 0 -> 0, 3 -> 2
    assert list(twoscale.nearest(np.arange(5), 2)) == [0, 1, 1, 2, 2]
    assert list(twoscale.nearest(np.arange(9), 4)) == [0, 0, 1, 1, 1, 1, 2, 2, 2]


def test_coarse_nb1_equals_fine_solve():
    # N_B = 1, z_C = z -> u_C = u
    nx, ny, nz = 4, 2, 2
    rho = np.random.default_rng(2).uniform(0.2, 1.0, nx * ny * nz)
    fixed, ld, lv = grid.cantilever_bc(nx, ny, nz)
    fc, ldc, lvc = twoscale.restrict_bc(nx, ny, nz, 1, fixed, ld, lv)
    edof = grid.element_dofs(nx, ny, nz)
    KE = fem.element_stiffness(0.3, 1.0)
    E = fem.simp(rho, 1.0, 1e-9, 3.0)
    K = fem.apply_bc(fem.assemble(edof, E, KE, fixed.size), fixed)
    f = grid.load_vector(fixed.size, ld, lv)
    fcv = grid.load_vector(fc.size, ldc, lvc)
    Kc = fem.apply_bc(fem.assemble(edof, fem.simp(twoscale.coarsen(rho, nx, ny, nz, 1), 1.0, 1e-9, 3.0),
                                   KE, fc.size), fc)
    assert np.allclose(solve.direct_solve(K, f), solve.direct_solve(Kc, fcv), rtol=1e-12, atol=0)


def test_coarse_uniform_compliance_scales_with_h():
    # a coarse solid cube of edge 2 (1 element, h = 2) is stiffer by the factor h: c = c(h=1)/2
    fixed, ld, lv = grid.cantilever_bc(1, 1, 1)
    edof = grid.element_dofs(1, 1, 1)
    f = grid.load_vector(24, ld, lv)
    cs = []
    for h in (1.0, 2.0):
        K = fem.apply_bc(fem.assemble(edof, np.ones(1), fem.element_stiffness(0.3, h), 24), fixed)
        cs.append(sens.compliance(f, solve.direct_solve(K, f)))
    assert abs(cs[1] - cs[0] / 2) <= 1e-13 * cs[0]
    assert abs(cs[0] - 43199 / 8400) <= 1e-12 * cs[0]
