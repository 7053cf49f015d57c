"""Mean device time of K_hat u (tomo_bench_apply, 200 back-to-back launches) at cfg3 and the
configs[4] grids; algorithmic bytes 16 N_dof + 8 N_e + N_n.
    python scripts/time_apply.py [grid ...]   (cfg3 | 4.0 .. 4.4; default cfg3 4.3 4.4)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
names = sys.argv[1:] or ["cfg3", "4.3", "4.4"]
lib = os.path.basename(os.environ.get("TOMO_LIB_PATH", "libtomo.so"))
for nm in names:
    if nm.startswith("cfg"):
        p = inputs.CONFIGS[nm]
        rho_np = inputs.density_for(nm)
    else:
        p = inputs.cfg4(int(nm.split(".")[1]))
        rho_np = inputs.density_void07(p)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.tensor(rho_np, dtype=torch.float64, device="cuda:0")
    # tomo_bench_apply applies the operator to the workspace's internal u: make it a realistic
    # field (a 20-iteration PCG iterate) rather than the zeros left by tomo_bind
    t.solve(rho, tol=0.0, max_iters=20)
    ms = min(t.bench_apply(rho, reps=200) for _ in range(3))
    b = 16 * p.n_dof + 8 * p.n_elem + p.n_node
    print(json.dumps({"lib": lib, "grid": [p.nx, p.ny, p.nz], "apply_us": round(ms * 1e3, 2),
                      "gbs": round(b / ms / 1e6, 1), "hbm_frac": round(b / ms / 1e6 / hbm, 4)}),
          flush=True)
    t.close()
