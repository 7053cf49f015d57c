"""GPU residual-vs-iteration curves (tomo_set_history) of the configs[4] void-0.7 solves, to
set beside the oracle's textbook PCG curves (scripts/oracle_runs/cfg4_void_curves.py;
VERDICT r1 item 1). Writes gpurun_out/void_curves_<tag>.json.
    python scripts/void_curves_gpu.py TAG [idx ...] [--exact-beta]   (idx 0..4; default 0 1 2)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

tag = sys.argv[1]
exact = "--exact-beta" in sys.argv
idxs = [int(a) for a in sys.argv[2:] if not a.startswith("--")] or [0, 1, 2]
out = {}
for idx in idxs:
    p = inputs.cfg4(idx)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    t.set_pcg_exact_beta(exact)
    rho = torch.tensor(inputs.density_void07(p), dtype=torch.float64, device="cuda:0")
    n = 50000
    h = t.set_history(n + 2)
    t.set_profiling(True)
    u, info = t.solve(rho, tol=1e-10, max_iters=n)
    pt = t.profile_times()
    c = t.compliance(u)
    rel = np.sqrt(h.cpu().numpy()[: info.iterations + 1]) / np.sqrt(1.0)  # ||f|| = 1 (cantilever, total -1 spread)
    fn = 1.0 / np.sqrt(p.ny + 1)  # ||f|| = sqrt((ny+1) (1/(ny+1))^2)
    rel = rel / fn
    keep = [(k, float(rel[k])) for k in range(len(rel)) if k < 50 or k % 50 == 0]
    out[p.name] = {"exact_beta": exact, "info": info.as_dict(), "compliance": c, "pcg_iter_ms": pt["k_a_ms"],
                   "curve_recursive": keep}
    print(p.name, info.as_dict(), c, pt, flush=True)
    t.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/void_curves_{tag}{'_exact' if exact else ''}.json", "w"))
