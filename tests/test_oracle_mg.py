"""Pins of the oracle's Galerkin multigrid (oracle/mg.py, reading R5): the 1-D
interpolation reproduces linear functions (so P maps coarse rigid-body modes to fine ones),
the Galerkin operator of an unconstrained grid annihilates the coarse rigid-body modes, and
MG-preconditioned CG reproduces the direct solve."""
import numpy as np
import pytest

from oracle import fem, grid, mg
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs


@pytest.mark.parametrize("n,pos", [(1, [0, 1]), (2, [0, 2]), (3, [0, 3]), (6, [0, 2, 4, 6]),
                                   (7, [0, 2, 4, 7])])
def test_coarse_positions(n, pos):
    assert list(mg.coarse_positions(n)) == pos


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11])
def test_prolong_1d_reproduces_linear(n):
    P = mg.prolong_1d(n).toarray()
    pos = mg.coarse_positions(n).astype(float)
    np.testing.assert_allclose(P.sum(axis=1), 1.0, rtol=0, atol=1e-15)  # constants
    np.testing.assert_allclose(P @ pos, np.arange(n + 1.0), rtol=0, atol=1e-14)  # linears


def _rigid_modes(n3):
    nx, ny, nz = n3
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    x, y, z = (a.ravel().astype(float) for a in (i, j, k))
    o, one = np.zeros_like(x), np.ones_like(x)
    modes = [(one, o, o), (o, one, o), (o, o, one), (-y, x, o), (o, -z, y), (z, o, -x)]
    return [np.stack(m, axis=1).ravel() for m in modes]


@pytest.mark.parametrize("n3", [(4, 3, 2), (5, 4, 3), (6, 6, 2)])
def test_galerkin_rigid_body_null_space(n3):
    nx, ny, nz = n3
    rng = np.random.default_rng(7)
    ne, _, ndof = grid.counts(nx, ny, nz)
    K = fem.assemble(grid.element_dofs(nx, ny, nz), rng.uniform(0.1, 1.0, ne),
                     fem.element_stiffness(0.3, 1.0), ndof)
    fixed = np.zeros(ndof, dtype=bool)
    A_c, Pm, fixed_c = mg.galerkin(K, n3, fixed)
    assert not fixed_c.any()
    nc = mg.coarse_elems(n3)
    scale = abs(A_c).max()
    for m_c, m_f in zip(_rigid_modes(nc), _rigid_modes(n3)):
        # P maps the coarse rigid mode (in coarse node coordinates scaled to fine positions)
        # onto the fine one; K annihilates it, so A_c does too
        pos = [mg.coarse_positions(n).astype(float) for n in n3]
        kk, jj, ii = np.meshgrid(pos[2], pos[1], pos[0], indexing="ij")
        x, y, z = ii.ravel(), jj.ravel(), kk.ravel()
        o, one = np.zeros_like(x), np.ones_like(x)
        coarse = {0: (one, o, o), 1: (o, one, o), 2: (o, o, one), 3: (-y, x, o),
                  4: (o, -z, y), 5: (z, o, -x)}
        idx = [np.allclose(m_f, r) for r in _rigid_modes(n3)].index(True)
        v = np.stack(coarse[idx], axis=1).ravel()
        np.testing.assert_allclose(Pm @ v, m_f, atol=1e-12)
        assert np.abs(A_c @ v).max() <= 1e-11 * scale * np.abs(v).max()


def test_galerkin_fixed_coarse_nodes_cantilever():
    p, _ = inputs.random_problem(6, 4, 4, seed=0)
    op = OracleProblem(p)
    fixed_c = mg.coarse_fixed(op.fixed, (6, 4, 4))
    # the clamped face x = 0 coarsens to the coarse face x = 0, all three components
    nc = mg.coarse_elems((6, 4, 4))
    f3 = fixed_c.reshape(nc[2] + 1, nc[1] + 1, nc[0] + 1, 3)
    assert f3[:, :, 0, :].all() and not f3[:, :, 1:, :].any()


def test_mgpcg_matches_direct_cfg0():
    p = inputs.CONFIGS["cfg0"]
    rho = inputs.density_for("cfg0")
    op = OracleProblem(p)
    A = op.Khat(rho)
    levels = mg.hierarchy(A, (p.nx, p.ny, p.nz), op.fixed, 400)
    assert len(levels) >= 3
    u, k, rr = mg.mgpcg(levels, op.f, tol=1e-10, nu=2, omega=0.6)
    u_ref = op.solve_direct(rho)
    assert rr <= 1e-10 and k < 30  # measured 14 (Jacobi-PCG: 383)
    assert np.linalg.norm(u - u_ref) <= 1e-8 * np.linalg.norm(u_ref)
