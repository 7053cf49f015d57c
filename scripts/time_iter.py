"""Device time per PCG iteration of a fixed-length solve (tol 0, N iterations) at a config,
CUDA events around the whole tomo_solve on the bound stream (so kernel boundaries and the
loop's own overheads are included), best of 3.
    python scripts/time_iter.py [cfg] [iters]       (A/B knobs: TOMO_NO_PDL, TOMO_NO_GRAPH, TOMO_NO_SEP_RED)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
p = inputs.CONFIGS[cfg]
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
rho = torch.tensor(inputs.density_for(cfg), dtype=torch.float64, device="cuda:0")
t.solve(rho, tol=0.0, max_iters=iters)
best = None
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(t.stream):
        e0.record()
    t.solve(rho, tol=0.0, max_iters=iters)
    with torch.cuda.stream(t.stream):
        e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (iters + 1)
    best = us if best is None else min(best, us)
env = {k: os.environ[k] for k in ("TOMO_NO_PDL", "TOMO_NO_GRAPH", "TOMO_NO_SEP_RED") if k in os.environ}
print(json.dumps({"cfg": cfg, "iters": iters, "us_per_iteration": round(best, 2), "env": env,
                  "lib": os.path.basename(os.environ.get("TOMO_LIB_PATH", "libtomo.so"))}))
