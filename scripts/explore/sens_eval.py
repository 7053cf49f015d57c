"""tomo_evaluate with a short solve (for ncu -k regex:k_sens: the sensitivity of the evaluate path,
which reads the workspace's padded u; TOMO_SENS_DENSE=1 restores the dense + mask-byte reads).
    python scripts/explore/sens_eval.py [cfg3 | 4.x ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

for nm in sys.argv[1:] or ["cfg3"]:
    if nm.startswith("cfg"):
        p, rho_np = inputs.CONFIGS[nm], inputs.density_for(nm)
    else:
        p = inputs.cfg4(int(nm.split(".")[1]))
        rho_np = inputs.density_void07(p)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.tensor(rho_np, dtype=torch.float64, device="cuda:0")
    dc = t.zeros_elem()
    for _ in range(4):
        u, c, dcf, info = t.evaluate(rho, None, dc, None, tol=0.0, max_iters=30)
    torch.cuda.synchronize()
    print(nm, "ok", c, float(dc.sum()))
    t.close()
