"""GPU parity at the BASELINE.json configs' full sizes, in the launch configuration bench.py
times (the same context code path). Where the oracle cannot finish a full solve in seconds
(configs[3], [4]), the CUDA result is checked through properties the oracle computes one
pass at a time: the true residual of u_gpu under the oracle's own K_hat, the oracle's c and
dc evaluated at u_gpu, and operator parity."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import filt, oc as ooc, sens
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs, tomo
from paper_2104_12282_b200.loop import SimpLoop

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def cpu(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def ctx(p):
    return tomo.Tomo(tomo.params_from_problem(p), device=DEV)


# ------------------------------------------------------------------ configs[3], the metric
def test_cfg3_evaluation_residual_pins():
    p = inputs.CFG3
    rho = inputs.density_for("cfg3")
    t = ctx(p)
    u_g, c, dcf, info = t.evaluate(gpu(rho), tol=1e-10)
    assert info.converged >= 1
    u = cpu(u_g)
    op = OracleProblem(p, assemble=False)
    r = op.f - op.apply(rho, u)
    rel_true = np.linalg.norm(r) / np.linalg.norm(op.f)
    # the GPU's own true-residual report agrees with the oracle's operator; at the fp64 floor
    # (~8e-10 here) f - K u is rounding noise of two summation orders: 2% agreement
    assert abs(rel_true - info.rel_res_true) <= 2e-2 * rel_true + 1e-14
    assert rel_true <= 2e-9  # high contrast (1e9): the recursive 1e-10 drifts
    assert abs(c - sens.compliance(op.f, u)) <= 1e-12 * abs(c)
    dc_ref, ce = op.sensitivity(rho, u)
    dc = cpu(t.sensitivity(gpu(rho), u_g))
    assert rel(dc, dc_ref) <= 1e-12
    # energy identity f^T u = u^T K u up to u^T r
    E = op.E(rho)
    assert abs(float(np.dot(E, ce)) - c) <= 1e-8 * c
    P = filt.filter_matrix(p.nx, p.ny, p.nz, p.rmin)
    assert rel(cpu(dcf), filt.apply_transpose(P, dc_ref)) <= 1e-12


# ------------------------------------------------------------------ configs[2]
def _gold(name):
    path = os.path.join(GOLD, f"{name}_solve.npz")
    if not os.path.exists(path):
        pytest.fail(f"golden {path} missing (python scripts/make_golden.py {name})")
    with open(os.path.join(GOLD, f"{name}_solve.json")) as f:
        meta = json.load(f)
    return meta, np.load(path)


def test_cfg2_mbb_half_beam_against_tight_oracle():
    """configs[2] against the oracle's tight (1e-12) solution (reading A14). The GPU solves
    to 1e-10 as BJ states: c must agree to 1e-9 (quadratic in the energy error, App. A-6);
    u, dc and P^T dc to max(1e-8, 2 delta_floor) with delta_floor the ORACLE's own 1e-10 vs
    1e-12 difference (stored in the golden); at 1e-12 the GPU agrees to 1e-8 as well."""
    meta, gold = _gold("cfg2")
    df = meta["delta_floor"]
    p = inputs.CFG2
    rho = inputs.density_for("cfg2")
    t = ctx(p)
    u_g, c, dcf, info = t.evaluate(gpu(rho), tol=1e-10)
    assert info.converged >= 1
    # iteration count: the single-pass recurrence (reading R1) vs its CPU run, textbook beside
    k_sp = meta.get("pcg_single_pass_iters_1e-10")
    k_ref = k_sp if k_sp is not None else meta["pcg_iters_1e-10"]
    assert abs(info.iterations - k_ref) <= max(3, 0.02 * k_ref), (info.iterations, k_sp, meta["pcg_iters_1e-10"])
    assert abs(c - meta["c"]) <= 1e-9 * abs(meta["c"])
    assert rel(cpu(u_g), gold["u"]) <= max(1e-8, 2 * df["u"])
    dc = cpu(t.sensitivity(gpu(rho), u_g))
    assert rel(dc, gold["dc"]) <= max(1e-8, 2 * df["dc"])
    assert rel(cpu(dcf), gold["dcf"]) <= max(1e-8, 2 * df["dcf"])
    u12, info12 = t.solve(gpu(rho), tol=1e-12, max_iters=200000)
    assert info12.converged >= 1
    assert rel(cpu(u12), gold["u"]) <= 1e-8
    assert rel(cpu(t.sensitivity(gpu(rho), u12)), gold["dc"]) <= 1e-8
    # operator-level parity on the oracle's own u (no solver noise)
    dc_on_gold = cpu(t.sensitivity(gpu(rho), gpu(gold["u"])))
    assert rel(dc_on_gold, gold["dc"]) <= 1e-12


def test_cfg0_against_stored_tight_oracle_if_present():
    path = os.path.join(GOLD, "cfg0_solve.npz")
    if not os.path.exists(path):
        pytest.skip("cfg0 golden not generated (the direct-solve parity in test_gpu_parity covers cfg0)")
    meta, gold = _gold("cfg0")
    t = ctx(inputs.CFG0)
    rho = inputs.density_for("cfg0")
    u_g, c, dcf, info = t.evaluate(gpu(rho), tol=1e-10)
    assert abs(c - meta["c"]) <= 1e-9 * abs(meta["c"])
    assert rel(cpu(dcf), gold["dcf"]) <= 1e-8


# ------------------------------------------------------------------ configs[4] sweep
@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("variant", ["void07", "uniform"])
def test_cfg4_operator_parity(idx, variant):
    p = inputs.cfg4(idx)
    if p.n_elem > 2_000_000 and variant == "uniform":
        pytest.skip("largest grid checked once (void07) to bound the oracle's host memory")
    rho = inputs.density_void07(p) if variant == "void07" else inputs.density_uniform(p, 0.5)
    op = OracleProblem(p, assemble=False)
    u = inputs.random_vector(op.n_dof, seed=idx + 40)
    t = ctx(p)
    y = cpu(t.apply(gpu(rho), gpu(u)))
    assert rel(y, op.apply(rho, u)) <= 1e-13


def test_cfg4a_solve_residual_pins():
    """32^3 with 70% of the elements at E = Emin = 1e-9 (configs[4] void 0.7). At this
    contrast CG loses orthogonality and its iteration count depends on rounding (measured:
    GPU 11,211 vs the oracle's textbook PCG 15,310, both converged), so the pin is the true
    residual of u_gpu under the oracle's own K_hat, not the count."""
    p = inputs.cfg4(0)
    rho = inputs.density_void07(p)
    t = ctx(p)
    u_g, info = t.solve(gpu(rho), tol=1e-10)
    assert info.converged >= 1
    op = OracleProblem(p)
    u = cpu(u_g)
    r = op.f - op.Khat(rho) @ u
    rel_true = np.linalg.norm(r) / np.linalg.norm(op.f)
    # at 1e-10 the residual is rounding noise of f - K u in two summation orders: 2% agreement
    assert rel_true <= 2e-10 and abs(rel_true - info.rel_res_true) <= 2e-2 * rel_true
    assert abs(info.rel_res_recursive) <= 1e-10


# ------------------------------------------------------------------ configs[1]: 50-step loop
def _loop_gold():
    jp = os.path.join(GOLD, "cfg1_loop.json")
    if not os.path.exists(jp):
        pytest.fail("golden cfg1_loop.json missing (python scripts/make_golden.py cfg1)")
    with open(jp) as f:
        h = json.load(f)
    return h, np.load(os.path.join(GOLD, "cfg1_x.npz"))


def test_cfg1_loop_teacher_forced():
    h, xs = _loop_gold()
    p = inputs.CFG1
    t = ctx(p)
    loop = SimpLoop(t, volfrac=p.volfrac, move=p.move, eta=p.eta, tol=1e-10)
    for k in (0, 1, 10, 25, 49):
        xn, c, lam, steps, info = loop.step(gpu(xs[f"x{k}"]))
        assert abs(c - h["c"][k]) <= 1e-9 * h["c"][k], k
        assert abs(lam - h["lam"][k]) <= 1e-8 * h["lam"][k], k
        nxt = f"x{k + 1}"
        if nxt in xs:
            assert np.max(np.abs(cpu(xn) - xs[nxt])) <= 1e-6, k


def test_cfg1_loop_free_running_history():
    h, xs = _loop_gold()
    p = inputs.CFG1
    t = ctx(p)
    loop = SimpLoop(t, volfrac=p.volfrac, move=p.move, eta=p.eta, tol=1e-10)
    hist = loop.run(gpu(xs["x0"]), p.loop_iters)
    c_ref = np.array(h["c"])
    c = np.array(hist["c"])
    relc = np.abs(c - c_ref) / c_ref
    assert relc[0] <= 1e-9
    assert np.max(relc) <= 1e-8, relc  # measured 3.3e-11 (profiles/r2_configs_report.json)
    assert c[-1] < c[0]  # the standard optimiser makes progress
    assert np.max(np.abs(cpu(hist["x_final"]) - xs["x50"])) <= 1e-4


# ------------------------------------------------------------------ configs[3]: 20-step loop
def test_cfg3_loop_20_iterations():
    """BASELINE.json configs[3] loop (volfrac 0.3, reading A19): 20 SIMP/OC steps on the GPU.
    The oracle cannot solve 4.3M DOFs in seconds, so each step is pinned by invariants and
    the OC update is teacher-forced through the oracle's own oc_update on the GPU's
    gradient at the first and the last step."""
    p = inputs.CFG3
    t = ctx(p)
    loop = SimpLoop(t, volfrac=p.volfrac, move=p.move, eta=p.eta, tol=1e-10)
    x = gpu(inputs.density_for("cfg3"))
    P = filt.filter_matrix(p.nx, p.ny, p.nz, p.rmin)
    dv = filt.volume_gradient(P)
    target = p.volfrac * p.n_elem
    cs = []
    for k in range(p.loop_iters):
        xk = cpu(x)
        xn, c, lam, steps, info = loop.step(x)
        assert info.converged >= 1
        cs.append(c)
        xn_h = cpu(xn)
        assert xn_h.min() >= 0.0 and xn_h.max() <= 1.0
        assert np.max(np.abs(xn_h - xk)) <= p.move + 1e-15
        if steps > 0:  # reachable target: the volume constraint holds at the bisection's l2
            vol = float(dv @ xn_h)
            assert vol <= target * (1 + 1e-9) and vol >= target * (1 - 1e-6)
        if k in (0, p.loop_iters - 1):
            g = cpu(loop.g)
            xr, lr, sr, _ = ooc.oc_update(xk, g, dv, P, p.volfrac, p.move, p.eta)
            assert abs(lam - lr) <= 1e-12 * lr
            assert np.max(np.abs(xn_h - xr)) <= 1e-12
        x = xn
    assert cs[-1] < cs[0]  # progress


def test_cfg3_against_sampled_tight_oracle_if_present():
    """configs[3], the metric's workload, against the oracle's own tight (1e-12) solve
    (tests/golden/cfg3_sampled.json, written by scripts/make_golden.py cfg3 - about 1.5 h of
    host time, so sampled: c, the full-vector norms and seeded entries of u, dc, P^T dc).
    Bars (reading A14): c to 1e-9; u, dc, dcf to max(1e-8, 2 delta_floor) with delta_floor
    the ORACLE's own 1e-10 vs 1e-12 difference where the golden records it (else the GPU's
    own, with a 4x margin); the GPU at 1e-12 to 1e-8."""
    path = os.path.join(GOLD, "cfg3_sampled.json")
    if not os.path.exists(path):
        pytest.skip("cfg3 sampled golden not generated (python scripts/make_golden.py cfg3)")
    with open(path) as f:
        g = json.load(f)
    p = inputs.CFG3
    rho = gpu(inputs.density_for("cfg3"))
    t = ctx(p)
    idof, iel = np.array(g["dof_idx"]), np.array(g["elem_idx"])
    u12, c12, dcf12, info12 = t.evaluate(rho, tol=1e-12, max_iters=200000)
    assert info12.converged >= 1
    dc12 = cpu(t.sensitivity(rho, u12))
    u10, c10, dcf10, info10 = t.evaluate(rho, tol=1e-10)
    dc10 = cpu(t.sensitivity(rho, u10))
    su = lambda v: cpu(v)[idof] if isinstance(v, torch.Tensor) else v[idof]  # noqa: E731
    se = lambda v: cpu(v)[iel] if isinstance(v, torch.Tensor) else v[iel]  # noqa: E731
    gu, gdc, gdcf = np.array(g["u"]), np.array(g["dc"]), np.array(g["dcf"])
    assert abs(c12 - g["c"]) <= 1e-9 * abs(g["c"])
    assert abs(c10 - g["c"]) <= 1e-9 * abs(g["c"])
    df = g.get("delta_floor")
    for key, a12, a10, gold, full10, norm in (
            ("u", su(u12), su(u10), gu, cpu(u10), g["norm_u"]),
            ("dc", se(dc12), se(dc10), gdc, dc10, g["norm_dc"]),
            ("dcf", se(dcf12), se(dcf10), gdcf, cpu(dcf10), g["norm_dcf"])):
        bar = max(1e-8, 2 * df[key]) if df else max(1e-8, 4 * rel(a10, a12))
        assert rel(a12, gold) <= 1e-8, key
        assert rel(a10, gold) <= bar, (key, rel(a10, gold), bar)
        # the full-vector norm of the oracle's solution
        assert abs(np.linalg.norm(full10) - norm) <= bar * norm, key
    if g.get("pcg_iters_1e-10"):
        print(f"cfg3: GPU {info10.iterations} iterations, oracle textbook {g['pcg_iters_1e-10']}")
