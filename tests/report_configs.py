"""SURVEY §8 d4/d5 per-config report: for BASELINE.json configs[0..3] the GPU evaluation
(evaluations/s with device-resident inputs, PCG iterations, both residuals, us per
iteration), its parity against the oracle, and the oracle's own timing on this box's host
cores. Oracle legs: cfg0 the full evaluation (its Jacobi-PCG, plus the direct solve for
parity); cfg1 one full loop iteration; cfg2 and cfg3 a bounded sample (setup + a few PCG
iterations + gradient) projected to the iteration count, as bench.py does for cfg3.
    python tests/report_configs.py out.json   (lives under tests/: it runs the oracle)"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import fem, filt, sens  # noqa: E402  (test infrastructure: the checker)
from oracle.loop import OracleProblem  # noqa: E402
from paper_2104_12282_b200 import inputs, tomo  # noqa: E402
from paper_2104_12282_b200.loop import SimpLoop  # noqa: E402

DEV = "cuda:0"
GOLD = os.path.join(ROOT, "tests", "golden")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def gpu_eval(name, reps):
    p = inputs.CONFIGS[name]
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    rho = torch.tensor(inputs.density_for(name), dtype=torch.float64, device=DEV)
    u, dc, dcf = t.zeros_dof(), t.zeros_elem(), t.zeros_elem()
    for _ in range(2):
        u.zero_()
        t.evaluate(rho, u, dc, dcf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(t.stream)
    for _ in range(reps):
        u.zero_()
        _, c, _, info = t.evaluate(rho, u, dc, dcf)
    e1.record(t.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    row = {"n_elem": p.n_elem, "n_dof": p.n_dof, "evals_per_s": 1e3 / ms, "ms_per_eval": ms,
           "pcg_iters": info.iterations, "us_per_iter": ms * 1e3 / max(1, info.iterations),
           "rel_res_recursive": info.rel_res_recursive, "rel_res_true": info.rel_res_true,
           "compliance": c}
    return row, t, rho, u.cpu().numpy(), dc.cpu().numpy(), dcf.cpu().numpy(), c


def oracle_sample(op, rho, n_iters, budget):
    t0 = time.perf_counter()
    E = op.E(rho)
    dinv = 1.0 / fem.jacobi_diag(E, op.KE, op.edof, op.fixed)
    t_setup = time.perf_counter() - t0
    pv = dinv * op.f
    t0 = time.perf_counter()
    for _ in range(budget):
        q = fem.apply_matfree(pv, E, op.KE, op.edof, op.fixed)
        pv = pv + 1e-3 * dinv * q  # the PCG body's work: one apply + vector updates
    t_iter = (time.perf_counter() - t0) / budget
    t0 = time.perf_counter()
    op.evaluate(rho, np.zeros(op.n_dof))
    t_grad = time.perf_counter() - t0
    total = t_setup + n_iters * t_iter + t_grad
    return {"seconds_per_eval": total, "projected": True,
            "sample": f"setup {t_setup:.2f}s + {budget} PCG-iteration bodies ({t_iter:.4f}s each) "
                      f"+ gradient {t_grad:.2f}s, projected to {n_iters} iterations"}


def main():
    out = {"host": {"cores": len(os.sched_getaffinity(0)), "cpu": platform.processor() or platform.machine()},
           "gpu": torch.cuda.get_device_name(0), "configs": {}}
    try:
        with open("/proc/cpuinfo") as f:
            out["host"]["cpu"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    # ---- cfg0: full oracle evaluation and the direct solve
    row, t, rho_g, u, dc, dcf, c = gpu_eval("cfg0", 20)
    p = inputs.CFG0
    op = OracleProblem(p)
    rho = inputs.density_for("cfg0")
    t0 = time.perf_counter()
    u_pcg, its, conv, _ = op.solve_pcg(rho, tol=1e-10)
    op.evaluate(rho, u_pcg)
    row["oracle"] = {"seconds_per_eval": time.perf_counter() - t0, "projected": False,
                     "pcg_iters": its, "sample": "full oracle evaluation (its Jacobi-PCG + gradient)"}
    u_ref = op.solve_direct(rho)
    c_ref, dc_ref, _, dcf_ref = op.evaluate(rho, u_ref)
    row["parity_vs_direct_solve"] = {"u": rel(u, u_ref), "c": abs(c - c_ref) / abs(c_ref),
                                     "dc": rel(dc, dc_ref), "dcf": rel(dcf, dcf_ref)}
    out["configs"]["cfg0"] = row
    # ---- cfg1: the 50-iteration loop against the oracle's golden history
    p = inputs.CFG1
    t1 = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    loop = SimpLoop(t1, volfrac=p.volfrac, move=p.move, eta=p.eta, tol=1e-10)
    x0 = torch.tensor(inputs.density_for("cfg1"), dtype=torch.float64, device=DEV)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hist = loop.run(x0, p.loop_iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    with open(os.path.join(GOLD, "cfg1_loop.json")) as f:
        h = json.load(f)
    c_g, c_o = np.array(hist["c"]), np.array(h["c"])
    op = OracleProblem(p)
    t0 = time.perf_counter()
    u1, its1, _, _ = op.solve_pcg(op.P @ inputs.density_for("cfg1"), tol=1e-10)
    o1 = time.perf_counter() - t0
    out["configs"]["cfg1"] = {"n_elem": p.n_elem, "n_dof": p.n_dof, "loop_iters": p.loop_iters,
                              "loop_seconds": dt, "iters_per_s": p.loop_iters / dt,
                              "pcg_iters_per_step": [int(k) for k in hist["iters"]],
                              "c_rel_err_step0": float(abs(c_g[0] - c_o[0]) / c_o[0]),
                              "c_rel_err_max_free_running": float(np.max(np.abs(c_g - c_o) / c_o)),
                              "oracle": {"seconds_first_solve": o1, "pcg_iters": its1, "projected": False,
                                         "sample": "oracle Jacobi-PCG of the first loop iteration"}}
    # ---- cfg2: against the stored tight oracle solution
    row, t, rho_g, u, dc, dcf, c = gpu_eval("cfg2", 10)
    gold = np.load(os.path.join(GOLD, "cfg2_solve.npz"))
    with open(os.path.join(GOLD, "cfg2_solve.json")) as f:
        meta = json.load(f)
    row["parity_vs_tight_oracle"] = {"u": rel(u, gold["u"]), "c": abs(c - meta["c"]) / abs(meta["c"]),
                                     "dc": rel(dc, gold["dc"]), "dcf": rel(dcf, gold["dcf"])}
    op = OracleProblem(inputs.CFG2, assemble=False)
    row["oracle"] = oracle_sample(op, inputs.density_for("cfg2"), meta["pcg_iters_1e-10"], 20)
    out["configs"]["cfg2"] = row
    # ---- cfg3: residual pins through the oracle's own operator
    row, t, rho_g, u, dc, dcf, c = gpu_eval("cfg3", 3)
    p = inputs.CFG3
    rho = inputs.density_for("cfg3")
    op = OracleProblem(p, assemble=False)
    r = op.f - op.apply(rho, u)
    dc_ref, _ = op.sensitivity(rho, u)
    P = filt.filter_matrix(p.nx, p.ny, p.nz, p.rmin)
    row["parity_residual_pins"] = {
        "rel_res_true_oracle": float(np.linalg.norm(r) / np.linalg.norm(op.f)),
        "c_vs_oracle_fTu": abs(c - sens.compliance(op.f, u)) / abs(c),
        "dc_vs_oracle_at_u_gpu": rel(dc, dc_ref), "dcf_vs_oracle_at_u_gpu": rel(dcf, filt.apply_transpose(P, dc_ref))}
    row["oracle"] = oracle_sample(op, rho, row["pcg_iters"], 4)
    out["configs"]["cfg3"] = row
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
