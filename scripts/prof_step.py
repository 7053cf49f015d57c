"""Short profiling driver: a few fused PCG iterations, the sensitivity, the filter transpose
and one OC update at a BASELINE config, for ncu (run with TOMO_NO_GRAPH=1 so that the PCG
launches are ordinary kernel launches).
   python scripts/prof_step.py [cfg] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 12
p = inputs.CONFIGS[cfg]
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
rho = torch.tensor(inputs.density_for(cfg), dtype=torch.float64, device="cuda:0")
u, info = t.solve(rho, tol=1e-10, max_iters=iters)
dc = t.sensitivity(rho, u)
dcf = t.filter(dc, transpose=True)
dv = t.volume_grad()
xn, lam, steps = t.oc_update(rho, dcf, dv, 0.3)
torch.cuda.synchronize()
print("ok", cfg, info.as_dict(), lam, steps)
