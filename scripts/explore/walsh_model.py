"""Exploration (reading R1): why the CUDA path needs ~27% fewer Jacobi-PCG
iterations than every CPU variant on the configs[4] void-0.7 grid. Hypothesis: the kernel's
element operator works on corner DIFFERENCES (tensor-Walsh modes; the constant mode is never
formed into the product), so rigid translations are annihilated exactly, while assembled
CSR or dense-KE element products annihilate them only to rounding. This model applies K in
that factored form in numpy (w = T u_e, v = E D w with the constant-mode rows/columns of
D = T KE T^T / 64 removed, y_e = T^T v) and runs the oracle's textbook PCG with it.
    python scripts/explore/walsh_model.py [idx] [variant]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle import fem, grid, solve  # noqa: E402
from oracle.loop import OracleProblem  # noqa: E402
from paper_2104_12282_b200 import inputs  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
variant = sys.argv[2] if len(sys.argv) > 2 else "void07"
p = inputs.cfg4(idx)
rho = inputs.density_void07(p) if variant == "void07" else inputs.density_uniform(p, 0.5)
op = OracleProblem(p)
E = op.E(rho)
T = np.array([[np.prod([(1.0 if c[d] else -1.0) if (m >> d) & 1 else 1.0 for d in range(3)])
               for c in grid.CORNERS] for m in range(8)])           # T[m, a]
T3 = np.kron(T, np.eye(3))                                           # (mode, comp) x (corner, comp)
D = T3 @ op.KE @ T3.T / 64.0
Dr = D[3:, 3:]                                                       # modes 1..7 (no constant mode)
T3r = T3[3:, :]
edof = op.edof
fixed = op.fixed


def apply_walsh(u):
    uu = np.where(fixed, 0.0, u)
    ue = uu[edof]                                   # (N_e, 24)
    w = ue @ T3r.T                                  # differences: (N_e, 21)
    v = (w @ Dr.T) * E[:, None]
    ye = v @ T3r                                    # (N_e, 24)
    y = np.bincount(edof.ravel(), weights=ye.ravel(), minlength=u.size)
    return np.where(fixed, u, y)


dinv = 1.0 / fem.jacobi_diag(E, op.KE, edof, fixed)
t = time.time()
u, k, conv, rel = solve.pcg(apply_walsh, dinv, op.f, tol=1e-10, max_iters=60000)
print(json.dumps({"grid": p.name, "variant": variant, "apply": "factored (Walsh differences)",
                  "textbook_iters": k, "converged": bool(conv), "c": float(op.f @ u),
                  "seconds": time.time() - t}), flush=True)
