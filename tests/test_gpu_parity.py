"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs. Bars (BASELINE.json north_star): integer tables bit-exact; K_hat u
norm-wise <= 1e-13; u and dc <= 1e-8 (norm-wise, A14), compliance <= 1e-9."""
import numpy as np
import pytest
import torch

from oracle import fem, filt, grid, oc as ooc, sens
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs
from paper_2104_12282_b200 import tomo

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def cpu(t):
    return t.detach().cpu().numpy()


def ctx_for(p):
    return tomo.Tomo(tomo.params_from_problem(p), device=DEV)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


RAGGED = [(24, 12, 12, 1), (5, 3, 7, 1), (1, 1, 1, 1), (1, 6, 1, 1), (33, 9, 4, 1),
          (62, 15, 3, 2), (7, 2, 9, 2), (40, 20, 20, 1)]


# ------------------------------------------------------------------ integer tables (bit-exact)
@pytest.mark.parametrize("nx,ny,nz,bc", RAGGED)
def test_integer_tables_bit_exact(nx, ny, nz, bc):
    p = inputs.Problem("t", nx, ny, nz, bc=bc, rmin=2.0)
    t = ctx_for(p)
    assert np.array_equal(cpu(t.element_dofs()), grid.element_dofs(nx, ny, nz))
    fixed, ldofs, lvals = grid.bc_for(bc, nx, ny, nz)
    assert np.array_equal(cpu(t.fixed_mask()).astype(bool), fixed)
    d, v = t.loads()
    assert d == ldofs.tolist() and np.array_equal(np.array(v), lvals)
    assert np.array_equal(cpu(t.neighbor_counts()).astype(np.int64),
                          filt.neighbor_counts(nx, ny, nz, p.rmin))


# ------------------------------------------------------------------ operator
@pytest.mark.parametrize("nx,ny,nz,bc", RAGGED)
def test_apply_parity(nx, ny, nz, bc):
    p, rho = inputs.random_problem(nx, ny, nz, seed=nx * 100 + ny, bc=bc)
    op = OracleProblem(p)
    u = inputs.random_vector(op.n_dof, seed=7)
    t = ctx_for(p)
    y = cpu(t.apply(gpu(rho), gpu(u)))
    ref = op.apply(rho, u)
    assert rel(y, ref) <= 1e-13
    # fixed rows are identity rows exactly
    assert np.array_equal(y[op.fixed], u[op.fixed])


def test_apply_high_contrast_and_rigid_modes():
    # no BCs (EXPLICIT, nothing fixed): rigid translations and rotations are in the null space
    nx, ny, nz = 9, 7, 5
    p = tomo.Params(nx, ny, nz, bc=tomo.TOMO_BC_EXPLICIT)
    t = tomo.Tomo(p, device=DEV)
    _, n_n, n_dof = grid.counts(nx, ny, nz)
    kk, jj, ii = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    X = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], 1).astype(float)
    rho = np.random.default_rng(1).uniform(0, 1, nx * ny * nz) ** 3
    for mode in range(6):
        u = np.zeros((n_n, 3))
        if mode < 3:
            u[:, mode] = 1.0
        else:
            a, b = [(1, 2), (2, 0), (0, 1)][mode - 3]
            u[:, a] = -X[:, b]
            u[:, b] = X[:, a]
        y = cpu(t.apply(gpu(rho), gpu(u.ravel())))
        assert np.max(np.abs(y)) <= 1e-12 * (1 + np.max(np.abs(u)))


def test_apply_cfg3_full_size_sampled():
    """Full BASELINE size (configs[3]) in the launch configuration the bench uses."""
    p = inputs.CFG3
    rho = inputs.density_for("cfg3")
    op = OracleProblem(p, assemble=False)
    u = inputs.random_vector(op.n_dof, seed=11)
    t = ctx_for(p)
    y = cpu(t.apply(gpu(rho), gpu(u)))
    ref = op.apply(rho, u)
    assert rel(y, ref) <= 1e-13


def test_jacobi_parity():
    p, rho = inputs.random_problem(13, 6, 5, seed=3, bc=2)
    op = OracleProblem(p)
    t = ctx_for(p)
    dinv = cpu(t.jacobi(gpu(rho)))
    d_ref = fem.jacobi_diag(op.E(rho), op.KE, op.edof, op.fixed)
    free = ~op.fixed
    per_dof = np.repeat(dinv, 3)
    assert np.max(np.abs(per_dof[free] * d_ref[free] - 1.0)) <= 1e-14


# ------------------------------------------------------------------ solve + gradient, cfg0
@pytest.fixture(scope="module")
def cfg0():
    p = inputs.CFG0
    rho = inputs.density_for("cfg0")
    op = OracleProblem(p)
    u_ref = op.solve_direct(rho)
    _, its_ref, conv, _ = op.solve_pcg(rho, tol=1e-10)
    assert conv
    return p, rho, op, u_ref, its_ref


def test_cfg0_solve_parity(cfg0):
    p, rho, op, u_ref, its_ref = cfg0
    t = ctx_for(p)
    u, info = t.solve(gpu(rho), tol=1e-10)
    u = cpu(u)
    assert info.converged >= 1
    assert info.rel_res_true <= 2e-10
    assert abs(info.iterations - its_ref) <= max(2, 0.02 * its_ref)
    assert rel(u, u_ref) <= 1e-8
    c = t.compliance(gpu(u))
    c_ref = sens.compliance(op.f, u_ref)
    assert abs(c - c_ref) / abs(c_ref) <= 1e-9


def test_cfg0_gradient_parity(cfg0):
    p, rho, op, u_ref, _ = cfg0
    t = ctx_for(p)
    u_g, c, dcf, info = t.evaluate(gpu(rho), tol=1e-10)
    c_ref, dc_ref, ce_ref, dcf_ref = op.evaluate(rho, u_ref)
    assert abs(c - c_ref) / abs(c_ref) <= 1e-9
    dc, energy = t.sensitivity(gpu(rho), u_g, energy=True)
    assert rel(cpu(dc), dc_ref) <= 1e-8
    assert rel(cpu(dcf), dcf_ref) <= 1e-8
    # operator-level parity of the sensitivity on the same u (no solver noise)
    # (Walsh-basis w^T D w vs the oracle's dense u^T KE u: different summation order, so
    # rounding-level only)
    dc_same, _ = op.sensitivity(rho, cpu(u_g))
    assert rel(cpu(dc), dc_same) <= 1e-12
    # energy identity u^T K u = f^T u at convergence from x0 = 0 (App. A-6)
    assert abs(energy - c) / c <= 1e-9


def test_tiny_cantilever_golden():
    # 1x1x1 -> 43199/8400, 2x1x1 -> 5428044583/222192210 (exact rationals)
    for (nx, num, den) in [(1, 43199, 8400), (2, 5428044583, 222192210)]:
        p = inputs.Problem("g", nx, 1, 1)
        t = ctx_for(p)
        rho = gpu(np.ones(nx))
        u, info = t.solve(rho, tol=1e-14, max_iters=1000)
        c = t.compliance(u)
        assert abs(c - num / den) <= 1e-12 * num / den


# ------------------------------------------------------------------ filter, OC
@pytest.mark.parametrize("nx,ny,nz,rmin", [(24, 12, 12, 1.5), (9, 5, 4, 2.0), (13, 7, 8, 3.0),
                                           (1, 1, 1, 1.5), (4, 3, 2, 0.9),
                                           # tiled kernel: every specialised / runtime-radius
                                           # path, ragged tiles (32 x 8) and several z chunks
                                           (70, 19, 37, 3.0), (45, 17, 29, 1.5), (33, 9, 40, 2.0),
                                           (37, 11, 23, 1.8), (35, 10, 26, 2.5), (29, 13, 31, 3.7),
                                           (26, 12, 30, 4.5), (27, 11, 33, 5.5), (25, 10, 28, 6.5),
                                           (40, 18, 35, 7.2), (21, 12, 25, 8.5), (20, 11, 22, 9.5),
                                           (5, 40, 3, 3.0)])
def test_filter_parity(nx, ny, nz, rmin):
    p = inputs.Problem("f", nx, ny, nz, rmin=rmin)
    t = ctx_for(p)
    P = filt.filter_matrix(nx, ny, nz, rmin)
    x = np.random.default_rng(5).uniform(0, 1, nx * ny * nz)
    assert rel(cpu(t.filter(gpu(x))), filt.apply(P, x)) <= 1e-14
    assert rel(cpu(t.filter(gpu(x), transpose=True)), filt.apply_transpose(P, x)) <= 1e-14
    assert rel(cpu(t.volume_grad()), filt.volume_gradient(P)) <= 1e-14


def test_oc_parity_1000_random_instances():
    """SPEC.md l.636 (acceptance criterion 3: 1,000 random (z, g, dV) instances) through the
    k_oc kernel against oracle/oc.py: box and move limits, the volume target within 1e-6 when
    reachable, lambda to 1e-13 and x to 1e-12. The two sides sum the volume in different
    orders, so a bisection decision can flip where V(lm) is within rounding of the target
    (reading A17): every instance whose lambda differs is checked to be such a flip - the
    oracle's own volume at the GPU's lambda equals the target to 1e-12."""
    rng = np.random.default_rng(0)
    nx, ny, nz = 8, 6, 5
    p = inputs.Problem("o", nx, ny, nz, rmin=1.5)
    t = ctx_for(p)
    P = filt.filter_matrix(nx, ny, nz, 1.5)
    dv = filt.volume_gradient(P)
    dv_g = t.volume_grad()
    assert rel(cpu(dv_g), dv) <= 1e-14
    n = nx * ny * nz
    flips = unreachable = wide = 0
    for inst in range(1000):
        x = rng.uniform(0.0, 1.0, n)
        g = -rng.uniform(0, 1, n) ** 3 * 10 ** rng.uniform(-3, 3)
        if inst % 10 == 0:
            g[rng.integers(0, n, 5)] = 0.0  # zero drive on some elements
        vf = rng.uniform(0.05, 0.95)
        move = rng.choice([0.05, 0.2, 0.5])
        xn_ref, lam_ref, steps_ref, _ = ooc.oc_update(x, g, dv, P, vf, move, 0.5)
        xn, lam, steps = t.oc_update(gpu(x), gpu(g), dv_g, vf, move, 0.5)
        xh = cpu(xn)
        assert xh.min() >= 0.0 and xh.max() <= 1.0
        assert np.all(np.abs(xh - x) <= move * (1 + 1e-15))
        assert (steps < 0) == (steps_ref < 0)
        if steps > 0:
            assert abs(float(np.sum(P @ xh)) - vf * n) <= 1e-6 * vf * n
        else:
            unreachable += 1
        assert np.max(np.abs(xh - xn_ref)) <= 1e-12
        if lam != lam_ref:
            flips += 1
            # a flip is admissible only where the volume decision is at rounding level: the
            # oracle's own volume at the GPU's lambda meets the target to 1e-12. Where V(lambda)
            # is flat there (every element at a move limit) lambda itself is ill-determined
            # while x is not, so lambda is compared only when the volume is not flat.
            v_at = float(np.sum(P @ ooc.x_new(x, g, dv, lam, move, 0.5)))
            assert abs(v_at - vf * n) <= 1e-12 * vf * n, (inst, v_at, vf * n)
            if abs(lam - lam_ref) > 1e-13 * lam_ref:
                wide += 1
                v_ref_at = float(np.sum(P @ ooc.x_new(x, g, dv, lam_ref, move, 0.5)))
                assert abs(v_at - v_ref_at) <= 1e-12 * vf * n, (inst, lam, lam_ref)
    print(f"OC 1000 instances: {flips} lambda flips (all at rounding-level volume decisions; "
          f"{wide} on a flat V(lambda)), {unreachable} unreachable targets")
    assert flips <= 500 and wide <= 50


# ------------------------------------------------------------------ edges and errors
def test_zero_load_gives_zero_iterations():
    p = tomo.Params(3, 2, 2, bc=tomo.TOMO_BC_EXPLICIT, fixed_dofs=tuple(range(9)))
    t = tomo.Tomo(p, device=DEV)
    u, info = t.solve(gpu(np.full(12, 0.5)))
    assert info.iterations == 0 and float(u.abs().max()) == 0.0


def test_errors_domain_and_size():
    p = inputs.Problem("e", 3, 2, 2)
    t = ctx_for(p)
    with pytest.raises(tomo.TomoError) as ei:
        t.solve(gpu(np.full(12, 1.5)))
    assert ei.value.code == -2
    with pytest.raises(ValueError):
        t.solve(gpu(np.full(11, 0.5)))


def test_determinism_bitwise():
    p, rho = inputs.random_problem(20, 10, 6, seed=9)
    t = ctx_for(p)
    u1, i1 = t.solve(gpu(rho))
    u2, i2 = t.solve(gpu(rho))
    assert i1.iterations == i2.iterations
    assert torch.equal(u1, u2)
    d1 = t.sensitivity(gpu(rho), u1)
    d2 = t.sensitivity(gpu(rho), u2)
    assert torch.equal(d1, d2)


def test_evaluate_host_matches_device():
    p = inputs.CFG0
    rho = inputs.density_for("cfg0")
    t = ctx_for(p)
    _, c_d, dcf_d, info_d = t.evaluate(gpu(rho))
    rho_h = torch.tensor(rho).pin_memory()
    dcf_h = torch.zeros(p.n_elem, dtype=torch.float64).pin_memory()
    c_h, info_h = t.evaluate_host(rho_h, dcf_h)
    assert c_h == c_d and info_h.iterations == info_d.iterations
    assert torch.equal(dcf_h, dcf_d.cpu())
