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


# ---- second model: the kernel's exact factorisation. D has 45 non-zeros described by 7
# numbers; rigid rotations are annihilated exactly as well, since the shear
# modes enter only as sums w_x1 + w_y0 (zero for a rotation) and the normal modes only
# through the strain-like w_x0, w_y1, w_z2.
mode = {(1, 0, 0): 1, (0, 1, 0): 2, (0, 0, 1): 4, (1, 1, 0): 3, (1, 0, 1): 5, (0, 1, 1): 6,
        (1, 1, 1): 7}


def at(m, c, n, e):
    return D[3 * m + c, 3 * n + e]


mx, my, mz, mxy, mxz, myz, mxyz = 1, 2, 4, 3, 5, 6, 7
cb = at(mx, 0, my, 1)
camb = at(mx, 0, mx, 0) - cb
cg = at(mx, 1, mx, 1)
c1, c2, c3, c4 = at(mxy, 0, mxy, 0), at(mxy, 0, myz, 2), at(mxy, 2, mxz, 1), at(mxyz, 0, mxyz, 0)


def apply_core7(u):
    uu = np.where(fixed, 0.0, u)
    ue = uu[edof].reshape(-1, 8, 3)
    W = np.einsum("ma,eac->emc", T, ue)          # (N_e, 8 modes, 3 comps), differences
    wx, wy, wz, wxy, wxz, wyz, wxyz = (W[:, m, :] for m in (mx, my, mz, mxy, mxz, myz, mxyz))
    V = np.zeros_like(W)
    Bt = cb * (wx[:, 0] + wy[:, 1] + wz[:, 2])
    V[:, mx, 0] = camb * wx[:, 0] + Bt
    V[:, my, 1] = camb * wy[:, 1] + Bt
    V[:, mz, 2] = camb * wz[:, 2] + Bt
    sxy, sxz, syz = cg * (wx[:, 1] + wy[:, 0]), cg * (wx[:, 2] + wz[:, 0]), cg * (wy[:, 2] + wz[:, 1])
    V[:, mx, 1] = V[:, my, 0] = sxy
    V[:, mx, 2] = V[:, mz, 0] = sxz
    V[:, my, 2] = V[:, mz, 1] = syz
    s = wxy[:, 2] + wxz[:, 1] + wyz[:, 0]
    V[:, mxy, 2], V[:, mxz, 1], V[:, myz, 0] = c3 * (s + wxy[:, 2]), c3 * (s + wxz[:, 1]), c3 * (s + wyz[:, 0])
    V[:, mxy, 0] = c1 * wxy[:, 0] + c2 * wyz[:, 2]
    V[:, mxy, 1] = c1 * wxy[:, 1] + c2 * wxz[:, 2]
    V[:, mxz, 0] = c1 * wxz[:, 0] + c2 * wyz[:, 1]
    V[:, mxz, 2] = c1 * wxz[:, 2] + c2 * wxy[:, 1]
    V[:, myz, 1] = c1 * wyz[:, 1] + c2 * wxz[:, 0]
    V[:, myz, 2] = c1 * wyz[:, 2] + c2 * wxy[:, 0]
    V[:, mxyz, :] = c4 * wxyz
    ye = np.einsum("ma,emc->eac", T, V * E[:, None, None]).reshape(-1, 24)
    y = np.bincount(edof.ravel(), weights=ye.ravel(), minlength=u.size)
    return np.where(fixed, u, y)


t = time.time()
u2, k2, conv2, _ = solve.pcg(apply_core7, dinv, op.f, tol=1e-10, max_iters=60000)
print(json.dumps({"grid": p.name, "variant": variant, "apply": "7-coefficient core (the kernel's)",
                  "textbook_iters": k2, "converged": bool(conv2), "c": float(op.f @ u2),
                  "seconds": time.time() - t}), flush=True)
