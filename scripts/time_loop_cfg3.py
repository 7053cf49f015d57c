"""configs[3] 20-iteration SIMP/OC loop on the GPU: per-iteration PCG count,
compliance, Lagrange multiplier and wall time (every step through the C ABI).
    python scripts/time_loop_cfg3.py [out.json] [--warm]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402
from paper_2104_12282_b200.loop import SimpLoop  # noqa: E402

p = inputs.CFG3
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
warm = "--warm" in sys.argv
loop = SimpLoop(t, volfrac=p.volfrac, move=p.move, eta=p.eta, tol=1e-10, warm_start=warm)
x = torch.tensor(inputs.density_for("cfg3"), dtype=torch.float64, device="cuda:0")
rows = []
t_all = time.perf_counter()
for k in range(p.loop_iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, c, lam, steps, info = loop.step(x)
    torch.cuda.synchronize()
    rows.append({"k": k, "c": c, "lambda": lam, "oc_steps": steps, "pcg_iters": info.iterations,
                 "rel_res_true": info.rel_res_true, "seconds": time.perf_counter() - t0})
    print(json.dumps(rows[-1]), flush=True)
out = {"config": p.name, "warm_start": warm, "iterations": p.loop_iters, "seconds": time.perf_counter() - t_all, "rows": rows}
print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
outs = [a for a in sys.argv[1:] if not a.startswith("--")]
if outs:
    json.dump(out, open(outs[0], "w"), indent=1)
