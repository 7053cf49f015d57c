"""Write tests/golden fixtures from the ORACLE ONLY (no CUDA path is imported).

  python scripts/make_golden.py cfg1   # 50-iteration SIMP/OC loop history (BASELINE configs[1])
  python scripts/make_golden.py cfg2   # tight oracle solve of the MBB half-beam (configs[2])
  python scripts/make_golden.py cfg0   # tight oracle solve of configs[0]

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


if __name__ == "__main__":
    for a in sys.argv[1:]:
        cfg1() if a == "cfg1" else tight(a)
