"""Residual-vs-iteration curves of the ORACLE's textbook Jacobi-PCG (oracle/solve.py) on the
configs[4] void-0.7 grids. Calls only oracle/ and inputs; writes
tests/golden/cfg4_void_oracle_<grid>.json (curves, iteration counts, compliance) and, where a
direct solve fits, the tight solution's compliance.

usage: python scripts/oracle_runs/cfg4_void_curves.py a|b [max_iters] [--direct]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import fem, solve  # noqa: E402
from oracle.loop import OracleProblem  # noqa: E402
from paper_2104_12282_b200 import inputs  # noqa: E402

idx = "abcde".index(sys.argv[1])
max_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
p = inputs.cfg4(idx)
rho = inputs.density_void07(p)
op = OracleProblem(p)
E = op.E(rho)
A = fem.apply_bc(fem.assemble(op.edof, E, op.KE, op.n_dof), op.fixed)
dinv = 1.0 / fem.jacobi_diag(E, op.KE, op.edof, op.fixed)
fn = np.linalg.norm(op.f)
curve = []


def cb(k, rel):
    if k % 50 == 0 or k < 50:
        curve.append((k, rel))


out = {"grid": [p.nx, p.ny, p.nz], "n_dof": op.n_dof, "max_iters": max_iters}
t0 = time.time()
u, k, conv, rel = solve.pcg(A.__matmul__, dinv, op.f, tol=1e-10, max_iters=max_iters, callback=cb)
out["pcg_1e-10"] = {"iterations": k, "converged": bool(conv), "rel_res_recursive": rel,
                     "rel_res_true": float(np.linalg.norm(op.f - A @ u) / fn),
                     "compliance": float(op.f @ u), "seconds": time.time() - t0}
out["curve_recursive"] = curve
print(json.dumps(out["pcg_1e-10"]), flush=True)
if "--direct" in sys.argv:
    t0 = time.time()
    ud = solve.direct_solve(A, op.f)
    out["direct"] = {"compliance": float(op.f @ ud),
                     "rel_res_true": float(np.linalg.norm(op.f - A @ ud) / fn),
                     "u_rel_err_pcg": float(np.linalg.norm(u - ud) / np.linalg.norm(ud)),
                     "seconds": time.time() - t0}
    print(json.dumps(out["direct"]), flush=True)
dst = os.path.join(os.path.dirname(__file__), "..", "..", "profiles",
                   f"r2_void_curves_oracle_cfg4{sys.argv[1]}.json")
with open(dst, "w") as fh:
    json.dump(out, fh, indent=1)
