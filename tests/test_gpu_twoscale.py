"""GPU parity of the two-scale coarse path (
SPEC.md l.364-391) against oracle/twoscale.py."""
import numpy as np
import pytest
import torch

from oracle import fem, grid, sens, solve, twoscale
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs, tomo

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def cpu(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("dims,nb", [((24, 12, 12), 2), ((24, 12, 12), 4), ((8, 6, 4), 1),
                                     ((224, 112, 56), 4), ((9, 6, 3), 3)])
def test_coarsen_parity(dims, nb):
    p = inputs.Problem("c", *dims)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    z = np.random.default_rng(sum(dims)).uniform(0, 1, p.n_elem)
    zc = cpu(t.coarsen(gpu(z), nb))
    ref = twoscale.coarsen(z, *dims, nb)
    assert np.max(np.abs(zc - ref)) <= 1e-15 * np.max(np.abs(ref)) * 4


@pytest.mark.parametrize("dims,bc,nb", [((24, 12, 12), 1, 2), ((12, 8, 8), 2, 2), ((24, 12, 12), 1, 4)])
def test_coarse_bc_mask_bit_exact(dims, bc, nb):
    p = inputs.Problem("c", *dims, bc=bc)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    tc = t.coarse(nb)
    fixed, ld, lv = grid.bc_for(bc, *dims)
    fc, _, _ = twoscale.restrict_bc(*dims, nb, fixed, ld, lv)
    assert np.array_equal(cpu(tc.fixed_mask()).astype(bool), fc)


def _oracle_coarse(dims, bc, nb, rho):
    fixed, ld, lv = grid.bc_for(bc, *dims)
    fc, ldc, lvc = twoscale.restrict_bc(*dims, nb, fixed, ld, lv)
    cd = tuple(d // nb for d in dims)
    zc = twoscale.coarsen(rho, *dims, nb)
    edof = grid.element_dofs(*cd)
    KE = fem.element_stiffness(0.3, float(nb))
    K = fem.apply_bc(fem.assemble(edof, fem.simp(zc, 1.0, 1e-9, 3.0), KE, fc.size), fc)
    f = grid.load_vector(fc.size, ldc, lvc)
    return zc, K, f


def test_coarse_solve_cfg0_nb2_against_direct():
    dims, bc, nb = (24, 12, 12), 1, 2
    rho = inputs.density_for("cfg0")
    t = tomo.Tomo(tomo.params_from_problem(inputs.CFG0), device=DEV)
    tc = t.coarse(nb)
    zc_g = t.coarsen(gpu(rho), nb)
    uc, info = tc.solve(zc_g, tol=1e-10)
    zc, K, f = _oracle_coarse(dims, bc, nb, rho)
    u_ref = solve.direct_solve(K, f)
    assert info.converged >= 1
    assert rel(cpu(uc), u_ref) <= 1e-8
    c_ref = sens.compliance(f, u_ref)
    assert abs(tc.compliance(uc) - c_ref) <= 1e-9 * abs(c_ref)


def test_coarse_nb1_equals_fine():
    p, rho = inputs.random_problem(10, 6, 4, seed=4)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    tc = t.coarse(1)
    u, _ = t.solve(gpu(rho), tol=1e-12)
    uc, _ = tc.solve(t.coarsen(gpu(rho), 1), tol=1e-12)
    assert rel(cpu(uc), cpu(u)) <= 1e-10


def test_coarse_cfg3_nb4_residual_pins():
    """configs[3] at N_B = 4 (56 x 28 x 14 coarse elements, edge 4): the coarse solve of
    every two-scale iteration. Pins: the oracle's coarse K_hat applied to u_C."""
    dims, bc, nb = (224, 112, 56), 1, 4
    rho = inputs.density_for("cfg3")
    t = tomo.Tomo(tomo.params_from_problem(inputs.CFG3), device=DEV)
    tc = t.coarse(nb)
    uc, info = tc.solve(t.coarsen(gpu(rho), nb), tol=1e-10)
    assert info.converged >= 1
    zc, K, f = _oracle_coarse(dims, bc, nb, rho)
    u = cpu(uc)
    r = np.linalg.norm(f - K @ u) / np.linalg.norm(f)
    assert r <= 2e-9 and abs(r - info.rel_res_true) <= 2e-2 * r
    assert abs(tc.compliance(uc) - sens.compliance(f, u)) <= 1e-12 * abs(sens.compliance(f, u))
