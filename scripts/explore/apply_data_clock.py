"""K_hat u at cfg3: is the bench's 33-35 us (vs time_apply's 31 us) the data or the clock?
Times tomo_bench_apply on (a) a 20-iteration PCG iterate, (b) the converged solution right after
the solve, (c) the converged solution after a 5 s pause (clocks recovered), with SM clocks."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402


def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()


p = inputs.CONFIGS["cfg3"]
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
rho = torch.tensor(inputs.density_for("cfg3"), dtype=torch.float64, device="cuda:0")
t.solve(rho, tol=0.0, max_iters=20)
a = min(t.bench_apply(rho, reps=200) for _ in range(3))
print(json.dumps({"u": "20-iteration iterate", "apply_us": round(a * 1e3, 2), "clk": clk()}), flush=True)
t.solve(rho, tol=1e-10)
b = min(t.bench_apply(rho, reps=200) for _ in range(3))
print(json.dumps({"u": "converged, right after the solve", "apply_us": round(b * 1e3, 2), "clk": clk()}), flush=True)
time.sleep(5)
c = min(t.bench_apply(rho, reps=200) for _ in range(3))
print(json.dumps({"u": "converged, after a 5 s pause", "apply_us": round(c * 1e3, 2), "clk": clk()}), flush=True)
for _ in range(3):
    t.solve(rho, tol=1e-10)
d = min(t.bench_apply(rho, reps=200) for _ in range(3))
print(json.dumps({"u": "converged, after 3 more solves", "apply_us": round(d * 1e3, 2), "clk": clk()}), flush=True)
