"""configs[4] sweep (BASELINE.json): K_hat u applications/s, DOF-updates/s, GB/s and % of the
HBM roofline of the operator kernel, and PCG iterations / time per iteration per solve, for
grids 32^3 .. 256x128x128 at void fraction 0.7 (Emin = 1e-9) and uniform 0.5.
    python scripts/sweep_cfg4.py [out.json] [--no-solve]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_12282_b200 import inputs, tomo  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else None
solve = "--no-solve" not in sys.argv
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = []
for idx in range(5):
    p = inputs.cfg4(idx)
    t = tomo.Tomo(tomo.params_from_problem(p), device="cuda:0")
    gf, _ = t.bench_dfma()
    for variant in ("void07", "uniform"):
        rho_np = inputs.density_void07(p) if variant == "void07" else inputs.density_uniform(p, 0.5)
        rho = torch.tensor(rho_np, dtype=torch.float64, device="cuda:0")
        # tomo_bench_apply applies the operator to the workspace's internal u: make it a
        # realistic field (a 20-iteration PCG iterate) rather than the zeros left by tomo_bind
        t.solve(rho, tol=0.0, max_iters=20)
        ms = t.bench_apply(rho, reps=100)
        # algorithmic bytes of K_hat u: read u, write y (8 B/DOF each), E (8 B/elem), mask (1 B/node)
        b = 16 * p.n_dof + 8 * p.n_elem + p.n_node
        flops = 213 * p.n_elem
        row = {"grid": [p.nx, p.ny, p.nz], "variant": variant, "n_elem": p.n_elem, "n_dof": p.n_dof,
               "apply_ms": ms, "applies_per_s": 1e3 / ms, "dof_updates_per_s": p.n_dof * 1e3 / ms,
               "alg_bytes": b, "gbs": b / ms / 1e6, "hbm_frac": b / ms / 1e6 / hbm,
               "gflops": flops / ms / 1e6, "fp64_frac": flops / ms / 1e6 / gf}
        if solve and p.n_elem <= 5_000_000:
            t.set_profiling(True)
            u, info = t.solve(rho, tol=1e-10, max_iters=50000)
            pt = t.profile_times()
            t.set_profiling(False)
            bi = 8 * (8 * p.n_dof + p.n_node + p.n_elem) + p.n_node
            row.update({"pcg_iters": info.iterations, "converged": info.converged,
                        "rel_res_true": info.rel_res_true, "pcg_iter_ms": pt["k_a_ms"],
                        "pcg_iter_gbs": bi / pt["k_a_ms"] / 1e6 if pt["k_a_ms"] else None,
                        "pcg_iter_hbm_frac": bi / pt["k_a_ms"] / 1e6 / hbm if pt["k_a_ms"] else None})
        rows.append(row)
        print(json.dumps(row), flush=True)
    t.close()
if out:
    json.dump({"hbm_gbs": hbm, "rows": rows}, open(out, "w"), indent=1)
