"""State solve K_hat u = f (oracle; test infrastructure only).

Cites: PAPER:184 ("one needs to first solve u through K(z)u - f = 0 ...
Iterative solvers such as preconditioned conjugate gradient (PCG) and
multi-grid methods are typically used"); PAPER:240 ("PCG method with the Jacobi
preconditioner"); SPEC:169-177 [OP pcg]; SPEC:178-186 [OP dense_solve];
SURVEY §8 a4/a5 and reading A11 (stopping rule ||r_k||_2 <= tol ||f||_2 on the
recursive residual, x0 given, k = number of K p products).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class Breakdown(RuntimeError):
    pass


def direct_solve(Khat, f):
    """The plain definition u = K_hat^{-1} f, by sparse LU (SuperLU, symmetric ordering)."""
    lu = spla.splu(sp.csc_matrix(Khat), permc_spec="MMD_AT_PLUS_A")
    return lu.solve(f)


def pcg(apply_A, dinv, f, x0=None, tol=1e-10, max_iters=100000, callback=None,
        callback_u=None):
    """Textbook Jacobi-preconditioned CG, in the order of SURVEY §8 a4:

        r0 = f - A x0, z0 = D^-1 r0, p0 = z0
        loop: q = A p; alpha = (r.z)/(p.q); u += alpha p; r -= alpha q;
              stop if ||r|| <= tol ||f||; z = D^-1 r; beta = (r.z)_new/(r.z); p = z + beta p

    Returns (u, iterations, converged, ||r||/||f|| recursive). callback(k, rel) and
    callback_u(k, rel, u) are observation hooks (they must not modify u).
    pcg(identity) is pinned by tests (1 iteration), the 2x2 system of SPEC:176 too.
    """
    f = np.asarray(f, dtype=np.float64)
    u = np.zeros_like(f) if x0 is None else np.array(x0, dtype=np.float64)
    if np.any(dinv <= 0.0):
        raise ValueError("non-positive preconditioner (SPEC:173)")
    fnorm = np.linalg.norm(f)
    if fnorm == 0.0:
        return np.zeros_like(f), 0, True, 0.0
    r = f - apply_A(u) if np.any(u) else f.copy()
    rnorm = np.linalg.norm(r)
    if rnorm <= tol * fnorm:
        return u, 0, True, rnorm / fnorm
    z = dinv * r
    p = z.copy()
    rz = r @ z
    k = 0
    while k < max_iters:
        q = apply_A(p)
        k += 1
        pq = p @ q
        if not pq > 0.0:
            raise Breakdown(f"p^T A p = {pq} <= 0 at iteration {k} (SPEC:173)")
        alpha = rz / pq
        u += alpha * p
        r -= alpha * q
        rnorm = np.linalg.norm(r)
        if callback is not None:
            callback(k, rnorm / fnorm)
        if callback_u is not None:
            callback_u(k, rnorm / fnorm, u)
        if rnorm <= tol * fnorm:
            return u, k, True, rnorm / fnorm
        z = dinv * r
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return u, k, False, rnorm / fnorm
