"""The operator grid's schedule: the synchronised (tile, z-chunk) schedule
with one or several waves of blocks, and the balanced fallback, must give the same solution.
Chunk count and schedule are chosen at bind time; TOMO_ZCHUNKS / TOMO_SCHED force them."""
import json
import os

import numpy as np
import pytest
import torch

from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs, tomo

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ctx(p, monkeypatch, **env):
    for k in ("TOMO_ZCHUNKS", "TOMO_SCHED"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    return tomo.Tomo(tomo.params_from_problem(p), device=DEV)


@pytest.mark.parametrize("env", [{}, {"TOMO_ZCHUNKS": "1"}, {"TOMO_ZCHUNKS": "33"},
                                 {"TOMO_SCHED": "balanced"}])
def test_cfg2_solve_any_schedule(env, monkeypatch):
    """cfg2 (20 tiles, 33 node planes): 1 chunk = 20 blocks in one wave, 33 chunks = 660
    one-plane blocks in three waves, or the persistent balanced grid - each solution agrees
    with the oracle's tight (1e-12) golden to the BJ bar."""
    path = os.path.join(GOLD, "cfg2_solve.npz")
    if not os.path.exists(path):
        pytest.fail("golden cfg2_solve.npz missing (python scripts/make_golden.py cfg2)")
    gold = np.load(path)
    with open(os.path.join(GOLD, "cfg2_solve.json")) as f:
        meta = json.load(f)
    p = inputs.CFG2
    t = _ctx(p, monkeypatch, **env)
    rho = torch.tensor(inputs.density_for("cfg2"), dtype=torch.float64, device=DEV)
    u, info = t.solve(rho, tol=1e-12, max_iters=200000)
    assert info.converged >= 1
    u = u.cpu().numpy()
    assert np.linalg.norm(u - gold["u"]) <= 1e-8 * np.linalg.norm(gold["u"])
    # the count depends on rounding (partial sums grouped per block), not on the schedule
    assert abs(info.iterations - meta["pcg_iters_1e-12"]) <= 0.03 * meta["pcg_iters_1e-12"]


def test_cfg4e_multiwave_solve_residual_pin(monkeypatch):
    """256x128x128 (171 tiles): the chosen schedule is 5 chunks = 855 blocks in three waves
    of 296 resident slots. A short solve (tol 1e-3) is pinned by the true residual of u_gpu
    under the oracle's own operator, which must agree with the GPU's report."""
    p = inputs.cfg4(4)
    t = _ctx(p, monkeypatch)
    rho_np = inputs.density_uniform(p, 0.5)
    u_g, info = t.solve(torch.tensor(rho_np, dtype=torch.float64, device=DEV), tol=1e-3)
    assert info.converged >= 1 and info.iterations > 10
    op = OracleProblem(p, assemble=False)
    u = u_g.cpu().numpy()
    r = op.f - op.apply(rho_np, u)
    rel_true = np.linalg.norm(r) / np.linalg.norm(op.f)
    assert rel_true <= 1.01e-3
    assert abs(rel_true - info.rel_res_true) <= 1e-6 * rel_true
