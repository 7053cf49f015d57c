"""GPU parity of the multigrid-preconditioned CG: it
reaches the same u as the oracle's plain definition (direct or tight solve) on the same
inputs, with far fewer outer iterations than Jacobi-PCG."""
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


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_mg_cfg0_against_direct_solve():
    p = inputs.CFG0
    rho = inputs.density_for("cfg0")
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    t.mg_setup(3)
    u, info = t.solve_mg(gpu(rho), tol=1e-10)
    assert info.converged >= 1 and info.rel_res_true <= 2e-10
    op = OracleProblem(p)
    u_ref = op.solve_direct(rho)
    assert rel(u.cpu().numpy(), u_ref) <= 1e-8
    c_ref = float(op.f @ u_ref)
    assert abs(t.compliance(u) - c_ref) <= 1e-9 * abs(c_ref)
    _, ij = t.solve(gpu(rho), tol=1e-10)
    assert info.iterations * 5 < ij.iterations


def test_mg_cfg2_against_tight_oracle():
    meta = json.load(open(os.path.join(GOLD, "cfg2_solve.json")))
    gold = np.load(os.path.join(GOLD, "cfg2_solve.npz"))
    p = inputs.CFG2
    rho = inputs.density_for("cfg2")
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    t.mg_setup(5)
    u, info = t.solve_mg(gpu(rho), tol=1e-12)
    assert info.converged >= 1
    assert rel(u.cpu().numpy(), gold["u"]) <= 1e-8
    assert abs(t.compliance(u) - meta["c"]) <= 1e-9 * abs(meta["c"])
    assert info.iterations * 10 < meta["pcg_iters_1e-12"]


def test_mg_mbb_small_and_errors():
    p, rho = inputs.random_problem(16, 8, 8, seed=3, bc=inputs.BC_MBB_HALF)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    with pytest.raises(tomo.TomoError):
        t.solve_mg(gpu(rho))                     # not set up
    with pytest.raises(tomo.TomoError):
        t.mg_setup(5)                            # 16 x 8 x 8 halves only 3 times
    t.mg_setup(4)
    u, info = t.solve_mg(gpu(rho), tol=1e-11)
    op = OracleProblem(p)
    assert info.converged >= 1
    assert rel(u.cpu().numpy(), op.solve_direct(rho)) <= 1e-9


def test_mg_graph_and_host_batched_bit_identical():
    """The MG-CG loop as one CUDA graph (default) and as host-batched iterations
    (tomo_set_graph(ctx, 0)) run the same kernels on the device-resident scalars: same
    iteration count, bit-identical u."""
    p = inputs.CFG0
    rho = gpu(inputs.density_for("cfg0"))
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    t.mg_setup(3)
    u1, i1 = t.solve_mg(rho, tol=1e-10)
    t.set_graph(False)
    u2, i2 = t.solve_mg(rho, tol=1e-10)
    t.set_graph(True)
    u3, i3 = t.solve_mg(rho, tol=1e-10)
    assert i1.iterations == i2.iterations == i3.iterations and i1.converged >= 1
    assert torch.equal(u1, u2) and torch.equal(u1, u3)
