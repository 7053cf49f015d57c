"""GPU edge cases and generality of the path against the oracle: non-unit element size and
Poisson ratios (the Walsh core is derived per context), explicit BCs with partially fixed
nodes, non-integer SIMP exponents, OC with eta != 0.5 / unreachable targets, the paper-scale
filter radius (7.2 elements, 1551 taps), warm starts, the max-iteration exit and
bitwise determinism of a whole evaluation."""
import numpy as np
import pytest
import torch

from oracle import fem, filt, grid, oc as ooc, sens, solve
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


@pytest.mark.parametrize("nu,h", [(0.25, 1.0), (0.45, 2.5), (0.3, 0.1), (0.05, 1.0)])
def test_apply_material_and_element_size(nu, h):
    nx, ny, nz = 11, 7, 5
    p = inputs.Problem("m", nx, ny, nz, nu=nu, h=h)
    rho = np.random.default_rng(3).uniform(0.01, 1, p.n_elem)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u = inputs.random_vector(p.n_dof, 5)
    op = OracleProblem(p)
    assert rel(cpu(t.apply(gpu(rho), gpu(u))), op.apply(rho, u)) <= 1e-13


def test_explicit_partial_bcs_apply_and_solve():
    nx, ny, nz = 9, 5, 4
    _, n_n, n_dof = grid.counts(nx, ny, nz)
    rng = np.random.default_rng(11)
    fixed_nodes_face = [grid.node_id(0, j, k, nx, ny) for k in range(nz + 1) for j in range(ny + 1)]
    fixed = sorted({3 * n for n in fixed_nodes_face} | {3 * n + 2 for n in fixed_nodes_face[::2]} |
                   {3 * n + 1 for n in fixed_nodes_face[1::3]} | {int(d) for d in rng.choice(n_dof, 20)})
    fixed = [d for d in fixed if d % 3 != 2 or d // 3 not in (grid.node_id(nx, 2, nz, nx, ny),)]
    load_node = grid.node_id(nx, 2, nz, nx, ny)
    ldofs, lvals = (3 * load_node + 2, 3 * load_node), (-1.0, 0.25)
    fixed = [d for d in fixed if d not in ldofs]
    params = tomo.Params(nx, ny, nz, bc=tomo.TOMO_BC_EXPLICIT, fixed_dofs=tuple(fixed),
                         load_dofs=ldofs, load_vals=lvals)
    t = tomo.Tomo(params, device=DEV)
    fmask = np.zeros(n_dof, dtype=bool)
    fmask[fixed] = True
    assert np.array_equal(cpu(t.fixed_mask()).astype(bool), fmask)
    rho = rng.uniform(0.2, 1, nx * ny * nz)
    E = fem.simp(rho, 1.0, 1e-9, 3.0)
    KE = fem.element_stiffness(0.3)
    edof = grid.element_dofs(nx, ny, nz)
    u = rng.standard_normal(n_dof)
    assert rel(cpu(t.apply(gpu(rho), gpu(u))), fem.apply_matfree(u, E, KE, edof, fmask)) <= 1e-13
    K = fem.apply_bc(fem.assemble(edof, E, KE, n_dof), fmask)
    f = grid.load_vector(n_dof, np.array(ldofs), np.array(lvals))
    u_ref = solve.direct_solve(K, f)
    ug, info = t.solve(gpu(rho), tol=1e-12)
    assert info.converged >= 1 and rel(cpu(ug), u_ref) <= 1e-9
    assert abs(t.compliance(ug) - f @ u_ref) <= 1e-10 * abs(f @ u_ref)


@pytest.mark.parametrize("penal", [1.0, 2.5, 3.0, 4.0])
def test_simp_exponent_sensitivity(penal):
    p = inputs.Problem("s", 10, 5, 4, penal=penal)
    rho = np.random.default_rng(7).uniform(0.05, 1, p.n_elem)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    op = OracleProblem(p)
    u = inputs.random_vector(p.n_dof, 9)
    u[op.fixed] = 0.0
    dc_ref, ce_ref = op.sensitivity(rho, u)
    dc, energy = t.sensitivity(gpu(rho), gpu(u), energy=True)
    assert rel(cpu(dc), dc_ref) <= 1e-12
    assert abs(energy - float(op.E(rho) @ ce_ref)) <= 1e-12 * abs(energy)


@pytest.mark.parametrize("eta,move,vf", [(0.3, 0.1, 0.4), (0.5, 0.2, 0.02), (0.5, 0.2, 0.98), (0.7, 0.05, 0.3)])
def test_oc_eta_move_and_unreachable(eta, move, vf):
    nx, ny, nz = 8, 6, 4
    p = inputs.Problem("o", nx, ny, nz)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    P = filt.filter_matrix(nx, ny, nz, 1.5)
    dv = filt.volume_gradient(P)
    rng = np.random.default_rng(int(eta * 100))
    x = rng.uniform(0.2, 0.6, nx * ny * nz)
    g = -rng.uniform(0, 2, nx * ny * nz)
    xn_ref, lam_ref, steps_ref, _ = ooc.oc_update(x, g, dv, P, vf, move, eta)
    xn, lam, steps = t.oc_update(gpu(x), gpu(g), t.volume_grad(), vf, move, eta)
    assert (steps < 0) == (steps_ref < 0)
    assert abs(lam - lam_ref) <= 1e-13 * lam_ref
    assert np.max(np.abs(cpu(xn) - xn_ref)) <= 1e-12


def test_paper_scale_filter_radius():
    # R = 0.08 on the inferred Mesh 3 is 7.2 elements (1551 taps)
    nx, ny, nz = 20, 12, 10
    p = inputs.Problem("f", nx, ny, nz, rmin=7.2)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    assert t.n_taps == 1551
    P = filt.filter_matrix(nx, ny, nz, 7.2)
    x = np.random.default_rng(2).uniform(0, 1, nx * ny * nz)
    assert rel(cpu(t.filter(gpu(x))), P @ x) <= 1e-14
    assert rel(cpu(t.filter(gpu(x), transpose=True)), P.T @ x) <= 1e-14


def test_warm_start_and_max_iters():
    p, rho = inputs.random_problem(16, 8, 6, seed=5)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u_cold, i_cold = t.solve(gpu(rho), tol=1e-10)
    u0 = u_cold.clone() * (1 + 1e-6)
    u_warm, i_warm = t.solve(gpu(rho), u=u0, tol=1e-10)
    assert i_warm.converged >= 1 and i_warm.iterations < i_cold.iterations
    assert rel(cpu(u_warm), cpu(u_cold)) <= 1e-8
    u_cap, i_cap = t.solve(gpu(rho), tol=1e-14, max_iters=7)
    assert i_cap.iterations == 7 and i_cap.converged == 0  # not an error


def test_evaluation_and_oc_bitwise_deterministic():
    p = inputs.CFG0
    rho = gpu(inputs.density_for("cfg0"))
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    outs = []
    for _ in range(2):
        u, c, dcf, info = t.evaluate(rho)
        xn, lam, steps = t.oc_update(rho, dcf, t.volume_grad(), 0.3)
        outs.append((u.clone(), c, dcf.clone(), info.iterations, xn.clone(), lam, steps))
    a, b = outs
    assert torch.equal(a[0], b[0]) and a[1] == b[1] and torch.equal(a[2], b[2]) and a[3] == b[3]
    assert torch.equal(a[4], b[4]) and a[5] == b[5] and a[6] == b[6]


@pytest.mark.parametrize("dims", [(24, 12, 12), (31, 9, 7), (33, 8, 5)])
def test_evaluate_sensitivity_on_padded_u_matches_dense_path(dims, monkeypatch):
    """tomo_evaluate's sensitivity reads the workspace's padded row-SoA solution; the dense
    path (TOMO_SENS_DENSE, what tomo_sensitivity does with a caller's u) must give the same dc
    bit for bit, and both match the oracle on the returned u (ragged tiles included)."""
    p = inputs.Problem("s", *dims, rmin=1.5)
    rho_np = np.random.default_rng(11).uniform(0.05, 1.0, p.n_elem)
    rho = gpu(rho_np)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    dc_pad, dc_dense = t.zeros_elem(), t.zeros_elem()
    u, c, dcf, info = t.evaluate(rho, None, dc_pad, None)
    monkeypatch.setenv("TOMO_SENS_DENSE", "1")
    u2, c2, dcf2, info2 = t.evaluate(rho, None, dc_dense, None)
    monkeypatch.delenv("TOMO_SENS_DENSE")
    assert torch.equal(u, u2) and torch.equal(dc_pad, dc_dense) and torch.equal(dcf, dcf2)
    assert torch.equal(dc_pad, t.sensitivity(rho, u))
    op = OracleProblem(p)
    # same u on both sides; a solved u makes u_e^T KE u_e a difference of large nearly equal
    # displacements, so the two summation orders differ by a few 1e-12 (measured 3e-12 - 5e-12)
    assert rel(cpu(dc_pad), op.sensitivity(rho_np, cpu(u))[0]) <= 1e-10


def test_paper_scale_filter_on_mesh3_sampled():
    """SURVEY f3 at full size: the paper's R = 0.08 on the inferred Mesh 3 (180x90x90, 1.46M
    elements, 7.2 elements = 1551 taps). The oracle cannot form P here
    (2.3e9 entries), so P x and P^T v are checked at 80 seeded elements - corners, faces and
    the interior - against oracle.filt.filter_rows, element by element."""
    nx, ny, nz, rmin = 180, 90, 90, 7.2
    p = inputs.Problem("mesh3", nx, ny, nz, rmin=rmin)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    assert t.n_taps == 1551
    x = np.random.default_rng(21).uniform(0, 1, p.n_elem)
    rng = np.random.default_rng(22)
    corners = [i + nx * (j + ny * k) for i in (0, nx - 1) for j in (0, ny - 1) for k in (0, nz - 1)]
    elems = np.array(sorted(set(corners) | set(rng.integers(0, p.n_elem, 72).tolist())))
    fwd = cpu(t.filter(gpu(x)))[elems]
    tr = cpu(t.filter(gpu(x), transpose=True))[elems]
    ref_f = filt.filter_rows(nx, ny, nz, rmin, elems, x)
    ref_t = filt.filter_rows(nx, ny, nz, rmin, elems, x, transpose=True)
    assert np.max(np.abs(fwd - ref_f) / np.abs(ref_f)) <= 1e-13
    assert np.max(np.abs(tr - ref_t) / np.abs(ref_t)) <= 1e-13
