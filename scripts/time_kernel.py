"""Mean device time of the fused PCG launch at a config over a fixed number of iterations
(results are meaningless for timing-experiment builds; only the time is read).
    python scripts/time_kernel.py [cfg] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
p = inputs.CONFIGS[cfg]
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
rho = torch.tensor(inputs.density_for(cfg), dtype=torch.float64, device="cuda:0")
t.solve(rho, tol=0.0, max_iters=20)
t.set_profiling(True)
try:
    t.solve(rho, tol=0.0, max_iters=iters)
except tomo.TomoError:
    pass  # experiment builds may break the recurrence; only the timing matters
print(os.path.basename(os.environ.get("TOMO_LIB_PATH", "libtomo.so")), cfg, t.profile_times())
