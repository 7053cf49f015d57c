"""Sensitivity kernel time (tomo_sensitivity, mean of 20 launches, CUDA events on the bound
stream) at cfg3 and the configs[4] grids; roofline: bytes 8 N_dof + 16 N_e (+ N_n mask),
DP: the Walsh energy w^T D w (~100 DP instructions per element) at the measured rate.
    python scripts/time_sens.py [cfg3 | 4.x ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for nm in sys.argv[1:] or ["cfg3", "4.4"]:
    if nm.startswith("cfg"):
        p, rho_np = inputs.CONFIGS[nm], inputs.density_for(nm)
    else:
        p = inputs.cfg4(int(nm.split(".")[1]))
        rho_np = inputs.density_void07(p)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.tensor(rho_np, dtype=torch.float64, device="cuda:0")
    u = torch.randn(p.n_dof, dtype=torch.float64, device="cuda:0")
    dc = t.zeros_elem()
    for _ in range(3):
        t.sensitivity(rho, u, dc)
    torch.cuda.synchronize()
    with torch.cuda.stream(t.stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(t.stream)
        for _ in range(20):
            t.sensitivity(rho, u, dc)
        e1.record(t.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    b = 8 * p.n_dof + 16 * p.n_elem + p.n_node
    print(json.dumps({"grid": [p.nx, p.ny, p.nz], "sens_us": round(ms * 1e3, 2), "gbs": round(b / ms / 1e6, 1),
                      "hbm_frac": round(b / ms / 1e6 / hbm, 3)}), flush=True)
    t.close()
