"""MG-CG vs Jacobi-PCG: iterations, time, compliance agreement (exploration / timing)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

runs = [tuple([r.split(":")[0], int(r.split(":")[1])]) for r in os.environ.get("MG_RUNS", "cfg0:3,cfg2:4,cfg2:5,cfg3:3,cfg3:4").split(",")]
nu = int(os.environ.get("MG_NU", "2"))
om = float(os.environ.get("MG_OMEGA", "0.6"))
ci = int(os.environ.get("MG_CI", "200"))
ct = float(os.environ.get("MG_CT", "1e-3"))
for name, levels in runs:
    p = inputs.CONFIGS[name]
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    rho = torch.tensor(inputs.density_for(name), dtype=torch.float64, device="cuda:0")
    t.mg_setup(levels, nu=nu, omega=om, coarse_iters=ci, coarse_tol=ct)
    uj, ij = t.solve(rho, tol=1e-10)
    cj = t.compliance(uj)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        um, im = t.solve_mg(rho, tol=1e-10, max_iters=int(os.environ.get("MG_MAX", "600")))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        cm = t.compliance(um)
        du = float(torch.linalg.norm(um - uj) / torch.linalg.norm(uj))
        print(json.dumps({"cfg": name, "levels": levels, "nu": nu, "omega": om, "mg_iters": im.iterations,
                          "mg_converged": im.converged, "mg_rel_true": im.rel_res_true, "mg_s": dt,
                          "jac_iters": ij.iterations, "c_rel_diff": abs(cm - cj) / abs(cj), "u_rel_diff": du}), flush=True)
    except tomo.TomoError as ex:
        print(json.dumps({"cfg": name, "levels": levels, "error": str(ex)}), flush=True)
