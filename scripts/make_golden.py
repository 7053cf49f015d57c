"""Write tests/golden fixtures from the ORACLE ONLY (no CUDA path is imported).

  python scripts/make_golden.py cfg1   # 50-iteration SIMP/OC loop history (BASELINE configs[1])
  python scripts/make_golden.py cfg2   # tight oracle solve of the MBB half-beam (configs[2])
  python scripts/make_golden.py cfg0   # tight oracle solve of configs[0]
  python scripts/make_golden.py cfg3   # tight oracle solve of configs[3], sampled (about an hour)

The oracle solves with its own Jacobi-PCG to a relative residual of 1e-12 (reading A14:
tighter than the 1e-10 the parity runs use), from x0 = 0.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import filt  # noqa: E402
from oracle.loop import OracleProblem, simp_loop  # noqa: E402
from paper_2104_12282_b200 import inputs  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def cfg1():
    p = inputs.CFG1
    op = OracleProblem(p)
    x0 = inputs.density_for("cfg1")
    t = time.time()
    keep = (0, 1, 10, 25, 49)
    h = simp_loop(op, x0, p.loop_iters, tol=1e-12, record_x=True)
    out = {"citation": "oracle/loop.simp_loop on BASELINE.json configs[1] (48x24x24 cantilever, x0 = 0.3, "
                       "50 SIMP/OC iterations, move 0.2, eta 0.5, volfrac 0.3, rmin 1.5); oracle PCG tol 1e-12 "
                       "from x0 = 0 each iteration (readings A6, A12, A17, A18). Written by scripts/make_golden.py.",
           "c": h["c"], "lam": h["lam"], "steps": h["steps"], "pcg_iters": h["iters"],
           "seconds": time.time() - t}
    with open(os.path.join(GOLD, "cfg1_loop.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(GOLD, "cfg1_x.npz"), **{f"x{k}": h["x"][k] for k in keep},
                        x50=h["x_final"])
    print("cfg1 done", out["seconds"])


def tight(name):
    p = inputs.CONFIGS[name]
    rho = inputs.density_for(name)
    op = OracleProblem(p)
    t = time.time()
    u, its, conv, rel = op.solve_pcg(rho, tol=1e-12)
    _, its10, _, _ = op.solve_pcg(rho, tol=1e-10)
    c, dc, ce, dcf = op.evaluate(rho, u)
    meta = {"citation": f"oracle Jacobi-PCG (tol 1e-12, x0 = 0) on BASELINE.json {name}; c = f^T u (Eq. 4), "
                        "dc (Eq. 5 with (E0-Emin), reading A5), dcf = P^T dc. Written by scripts/make_golden.py.",
            "c": c, "pcg_iters_1e-12": its, "pcg_iters_1e-10": its10, "converged": bool(conv),
            "rel_res": rel, "seconds": time.time() - t}
    with open(os.path.join(GOLD, f"{name}_solve.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(GOLD, f"{name}_solve.npz"), u=u, dc=dc, dcf=dcf)
    print(name, "done", meta)


def cfg3_sampled(n_sample=4096, seed=33):
    """configs[3] (4.35M DOFs): the oracle's own Jacobi-PCG to 1e-12 from x0 = 0 (about an
    hour on 8-16 host cores), stored as c, the iteration count, the true residual, the
    full-vector norms and seeded samples of u, dc and P^T dc ('full u parity
    is run locally')."""
    p = inputs.CFG3
    rho = inputs.density_for("cfg3")
    op = OracleProblem(p, assemble=False)
    t = time.time()
    u, its, conv, rel = op.solve_pcg(rho, tol=1e-12, max_iters=200000, use_csr=False)
    r = op.f - op.apply(rho, u)
    rel_true = float(np.linalg.norm(r) / np.linalg.norm(op.f))
    c, dc, ce, dcf = op.evaluate(rho, u)
    rng = np.random.default_rng(seed)
    idof = np.sort(rng.choice(op.n_dof, n_sample, replace=False))
    iel = np.sort(rng.choice(op.n_e, n_sample, replace=False))
    meta = {"citation": "oracle Jacobi-PCG (tol 1e-12 recursive, x0 = 0, matrix-free apply) on BASELINE.json "
                        "configs[3]; c = f^T u (Eq. 4), dc (Eq. 5, reading A5), dcf = P^T dc; seeded samples. "
                        "Written by scripts/make_golden.py cfg3.",
            "c": float(c), "pcg_iters_1e-12": int(its), "converged": bool(conv), "rel_res_recursive": float(rel),
            "rel_res_true": rel_true, "norm_u": float(np.linalg.norm(u)), "norm_dc": float(np.linalg.norm(dc)),
            "norm_dcf": float(np.linalg.norm(dcf)), "seconds": time.time() - t,
            "dof_idx": idof.tolist(), "u": u[idof].tolist(), "elem_idx": iel.tolist(),
            "dc": dc[iel].tolist(), "dcf": dcf[iel].tolist()}
    with open(os.path.join(GOLD, "cfg3_sampled.json"), "w") as f:
        json.dump(meta, f)
    print("cfg3 done", {k: meta[k] for k in ("c", "pcg_iters_1e-12", "rel_res_true", "seconds")})


if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a == "cfg1":
            cfg1()
        elif a == "cfg3":
            cfg3_sampled()
        else:
            tight(a)
