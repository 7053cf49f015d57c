"""Debug driver: one apply and one short solve on small grids, CUDA errors surfaced per call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2104_12282_b200 import inputs, tomo
from oracle.loop import OracleProblem
for dims in [(24, 12, 12), (40, 20, 20), (64, 30, 10)]:
    p, rho = inputs.random_problem(*dims, seed=1)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    u = inputs.random_vector(p.n_dof, 3)
    try:
        y = t.apply(torch.tensor(rho, device="cuda:0"), torch.tensor(u, device="cuda:0"))
        torch.cuda.synchronize()
        ref = OracleProblem(p).apply(rho, u)
        print(dims, "apply rel err", np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref), flush=True)
    except Exception as ex:
        print(dims, "apply failed", ex, flush=True); raise
    try:
        uu, info = t.solve(torch.tensor(rho, device="cuda:0"), max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 5)
        print(dims, "solve", info.as_dict(), flush=True)
    except Exception as ex:
        print(dims, "solve failed", ex, flush=True); raise
