"""configs[4] full-solve parity (32^3 and 64^3, void fraction 0.7 and uniform
0.5, plus 128x64x64 and 192x96x96 uniform) through the C ABI against the ORACLE's tight solutions (its textbook Jacobi-PCG to
1e-12 from x0 = 0, tests/golden/cfg4*_solve.{json,npz} (32^3, full vectors) and
cfg4*_sampled.json (64^3 and larger: c, norms, seeded samples), scripts/make_golden.py).

Bars (reading A14): the GPU solves to 1e-10 as BASELINE.json states; c to 1e-9; u, dc to
max(1e-8, 2 delta_floor), delta_floor = the oracle's OWN 1e-10 solution against its 1e-12
one (stored in the golden). At the void-0.7 contrast (E = 1e-9 on 70% of the elements) the
energy norm CG minimises barely weights the void DOFs, so delta_floor(u) is ~3e-7 there
while dc and c stay at ~1e-11. Iteration counts (reading R1): the kernel runs the
single-pass reformulation, pinned to that recurrence's CPU run (oracle.solve.
pcg_single_pass) where recorded; the textbook count is reported beside it."""
import json
import os

import numpy as np
import pytest
import torch

from paper_2104_12282_b200 import inputs, tomo

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = [("cfg4a_uniform", 0, "uniform"), ("cfg4a_void07", 0, "void07"),
         ("cfg4b_uniform", 1, "uniform"), ("cfg4c_uniform", 2, "uniform"),
         ("cfg4d_uniform", 3, "uniform")]


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _gold(name):
    for suffix, sampled in (("_solve.json", False), ("_sampled.json", True)):
        path = os.path.join(GOLD, name + suffix)
        if os.path.exists(path):
            with open(path) as f:
                meta = json.load(f)
            vec = None if sampled else np.load(os.path.join(GOLD, name + "_solve.npz"))
            return meta, vec
    pytest.fail(f"golden for {name} missing (python scripts/make_golden.py cfg4:...)")


@pytest.mark.parametrize("name,idx,variant", CASES)
def test_cfg4_full_solve_parity(name, idx, variant):
    meta, vec = _gold(name)
    p = inputs.cfg4(idx)
    rho_np = inputs.density_void07(p) if variant == "void07" else inputs.density_uniform(p, 0.5)
    rho = gpu(rho_np)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u10, info = t.solve(rho, tol=1e-10, max_iters=100000)
    assert info.converged >= 1, info.as_dict()
    c10 = t.compliance(u10)
    dc10 = t.sensitivity(rho, u10).cpu().numpy()
    u10 = u10.cpu().numpy()
    if vec is not None:
        du, ddc = rel(u10, vec["u"]), rel(dc10, vec["dc"])
    else:
        du = rel(u10[np.array(meta["dof_idx"])], np.array(meta["u"]))
        ddc = rel(dc10[np.array(meta["elem_idx"])], np.array(meta["dc"]))
        # full-vector norms of the oracle's solution
        assert abs(np.linalg.norm(u10) - meta["norm_u"]) <= max(1e-8, 2 * meta["delta_floor"]["u"]) * meta["norm_u"]
        assert abs(np.linalg.norm(dc10) - meta["norm_dc"]) <= max(1e-8, 2 * meta["delta_floor"]["dc"]) * meta["norm_dc"]
    bar_u = max(1e-8, 2 * meta["delta_floor"]["u"])
    bar_dc = max(1e-8, 2 * meta["delta_floor"]["dc"])
    print(f"{name}: GPU {info.iterations} it (single-pass model "
          f"{meta.get('pcg_single_pass_iters_1e-10')}, textbook {meta['pcg_iters_1e-10']}), "
          f"c {abs(c10 - meta['c']) / abs(meta['c']):.1e}, u {du:.1e} (bar {bar_u:.1e}), "
          f"dc {ddc:.1e} (bar {bar_dc:.1e}), true res {info.rel_res_true:.2e}")
    assert abs(c10 - meta["c"]) <= 1e-9 * abs(meta["c"])
    assert du <= bar_u and ddc <= bar_dc
    k_sp = meta.get("pcg_single_pass_iters_1e-10") or (meta["pcg_iters_1e-10"] if variant == "uniform" else None)
    if k_sp is not None and variant == "uniform":
        # well conditioned: the kernel's recurrence reproduces its CPU run; at the void-0.7
        # contrast the count is a property of the finite-precision trajectory and is only
        # reported (reading R1: CPU variants 15,054-15,530, the GPU 11,205)
        assert abs(info.iterations - k_sp) <= max(3, 0.02 * k_sp), (info.iterations, k_sp)


def test_cfg4b_void07_at_the_tolerance_both_reach():
    """64^3 void 0.7: neither the oracle's textbook PCG (relative residual 7.5e-7 after 50,000
    iterations) nor the GPU (1.6e-8) reaches 1e-10 (reading R1), so parity is
    checked at the tightest tolerance both reach: t* = the tightest
    snapshot of the oracle's tolerance ladder (tests/golden/cfg4b_void07_ladder.json: its
    iterate at the first crossing of each decade and at the 55,000-iteration cap). The GPU
    solves to t*; c, u and dc (seeded samples, full-vector norms) are compared with the
    oracle's t* iterate. Both iterates carry an error of the size the oracle's own t* iterate
    shows against its cap iterate (delta): the bars are 4 delta (c: 4 delta_c, floors 1e-9 /
    1e-8 as A14)."""
    path = os.path.join(GOLD, "cfg4b_void07_ladder.json")
    if not os.path.exists(path):
        pytest.fail("golden cfg4b_void07_ladder.json missing (python scripts/make_golden.py ladder:1void07)")
    with open(path) as f:
        g = json.load(f)
    assert g["final"] is not None, "ladder run incomplete"
    tstar = min(g["snapshots"], key=float)
    snap, fin = g["snapshots"][tstar], g["final"]
    idof, iel = np.array(g["dof_idx"]), np.array(g["elem_idx"])
    d_u = rel(np.array(snap["u"]), np.array(fin["u"]))
    d_dc = rel(np.array(snap["dc"]), np.array(fin["dc"]))
    d_c = abs(snap["c"] - fin["c"]) / abs(fin["c"])
    p = inputs.cfg4(1)
    rho = gpu(inputs.density_void07(p))
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u, info = t.solve(rho, tol=float(tstar), max_iters=60000)
    assert info.converged >= 1, info.as_dict()
    c = t.compliance(u)
    dc = t.sensitivity(rho, u).cpu().numpy()
    u = u.cpu().numpy()
    eu, edc = rel(u[idof], np.array(snap["u"])), rel(dc[iel], np.array(snap["dc"]))
    ec = abs(c - snap["c"]) / abs(snap["c"])
    print(f"cfg4b void07 at t* = {tstar}: GPU {info.iterations} it (oracle {snap['iterations']}), "
          f"c {ec:.1e} (bar {max(1e-9, 4 * d_c):.1e}), u {eu:.1e} (bar {max(1e-8, 4 * d_u):.1e}), "
          f"dc {edc:.1e} (bar {max(1e-8, 4 * d_dc):.1e})")
    assert ec <= max(1e-9, 4 * d_c)
    assert eu <= max(1e-8, 4 * d_u) and edc <= max(1e-8, 4 * d_dc)
    assert abs(np.linalg.norm(u) - snap["norm_u"]) <= max(1e-8, 4 * d_u) * snap["norm_u"]
