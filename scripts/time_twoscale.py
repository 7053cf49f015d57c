"""SURVEY §8 f1 (two-scale coarse path, PAPER Alg. 1 lines 3-4, run at every ONSG iteration):
block-average the design over N_B^3 elements and solve the coarse problem K_C(z_C) u_C = f_C
with the same fused Jacobi-PCG kernel, at configs[3] for N_B = 2, 4, 8; device time per
coarse step (coarsen + solve from x0 = 0 to 1e-10) against the fine exact evaluation.
    python scripts/time_twoscale.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

p = inputs.CFG3
t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
z = torch.tensor(inputs.density_for("cfg3"), dtype=torch.float64, device="cuda:0")
rows = []
for nb in (2, 4, 8):
    tc = t.coarse(nb)
    zc = t.coarsen(z, nb)
    uc, info = tc.solve(zc, tol=1e-10)  # warm-up
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 5
    ev[0].record(t.stream)
    for _ in range(reps):
        zc = t.coarsen(z, nb, out=zc)
        uc.zero_()
        uc, info = tc.solve(zc, uc, tol=1e-10)
    ev[1].record(t.stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    rows.append({"nb": nb, "coarse_elems": zc.numel(), "coarse_dofs": tc.n_dof, "pcg_iters": info.iterations,
                 "converged": info.converged, "rel_res_true": info.rel_res_true, "ms_per_coarse_step": ms})
    print(json.dumps(rows[-1]), flush=True)
    tc.close()
out = {"config": p.name, "rows": rows}
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
