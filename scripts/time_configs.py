"""Evaluations/s per BASELINE config (device-resident inputs, x0 = 0, tol 1e-10): quick A/B tool.
    python scripts/time_configs.py [cfg0 cfg2 cfg3 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

for name in (sys.argv[1:] or ["cfg0", "cfg2", "cfg3"]):
    p = inputs.CONFIGS[name]
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.tensor(inputs.density_for(name), dtype=torch.float64, device="cuda:0")
    u = t.zeros_dof()
    dcf = t.zeros_elem()
    for _ in range(2):
        u.zero_()
        t.evaluate(rho, u, None, dcf)
    torch.cuda.synchronize()
    n = 3 if p.n_elem > 1e6 else 10
    t0 = time.perf_counter()
    for _ in range(n):
        u.zero_()
        _, c, _, info = t.evaluate(rho, u, None, dcf)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(json.dumps({"cfg": name, "evals_per_s": 1 / dt, "ms_per_eval": dt * 1e3, "pcg_iters": info.iterations,
                      "us_per_iter": dt * 1e6 / max(1, info.iterations), "c": c,
                      "graph": not bool(os.environ.get("TOMO_NO_GRAPH"))}), flush=True)
