"""Two contexts on two CUDA streams at once (the ABI's per-context state, SURVEY §8 b:
"not thread-safe; one per problem", every call enqueued on the bound stream): results are
bitwise those of each context run alone, and the replicas path of bench.py (one context per
rank) therefore needs no cross-context synchronisation."""
import numpy as np
import pytest
import torch

from paper_2104_12282_b200 import inputs, tomo

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _run(p, rho_np, stream=None):
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV, stream=stream)
    rho = torch.tensor(rho_np, dtype=torch.float64, device=DEV)
    u, c, dcf, info = t.evaluate(rho, tol=1e-10)
    torch.cuda.synchronize()
    return t, u.cpu().numpy(), c, dcf.cpu().numpy(), info.iterations


def test_two_contexts_two_streams_bitwise():
    pa, ra = inputs.CFG0, inputs.density_for("cfg0")
    pb, rb = inputs.random_problem(17, 9, 6, seed=5)
    _, ua, ca, da, ka = _run(pa, ra)
    _, ub, cb, db, kb = _run(pb, rb)
    sa, sb = torch.cuda.Stream(device=DEV), torch.cuda.Stream(device=DEV)
    ta = tomo.Tomo(tomo.params_from_problem(pa), device=DEV, stream=sa)
    tb = tomo.Tomo(tomo.params_from_problem(pb), device=DEV, stream=sb)
    rga = torch.tensor(ra, dtype=torch.float64, device=DEV)
    rgb = torch.tensor(rb, dtype=torch.float64, device=DEV)
    torch.cuda.synchronize()
    # interleave the two evaluations (each call synchronises only its own stream)
    out = []
    for _ in range(3):
        out.append((ta.evaluate(rga, tol=1e-10), tb.evaluate(rgb, tol=1e-10)))
    torch.cuda.synchronize()
    for (ua2, ca2, da2, ia), (ub2, cb2, db2, ib) in out:
        assert np.array_equal(ua2.cpu().numpy(), ua) and ca2 == ca and ia.iterations == ka
        assert np.array_equal(da2.cpu().numpy(), da)
        assert np.array_equal(ub2.cpu().numpy(), ub) and cb2 == cb and ib.iterations == kb
        assert np.array_equal(db2.cpu().numpy(), db)
