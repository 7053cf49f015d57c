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


def pcg_single_pass(apply_A, dinv, f, x0=None, tol=1e-10, max_iters=100000, callback=None):
    """The single-reduction reformulation of the same Jacobi-PCG (reading R1; the
    recurrence the fused CUDA kernel runs, restated here from that description - no code is
    shared). Mathematically it produces the iterates of pcg() above: with q = A p,
    r_{k+1}.z_{k+1} = r.z - 2 alpha z.q + alpha^2 q.D^-1.q, so beta needs no second
    reduction. "Launch" k forms
        r_k = r_{k-1} - alpha_{k-1} q_{k-1},  z_k = D^-1 r_k,  p_k = z_k + beta_{k-1} p_{k-1},
        u_k = u_{k-1} + alpha_{k-1} p_{k-1},  q_k = A p_k,
    reduces p.q, r.z, r.r, z.q, q.D^-1.q, stops when ||r_k|| <= tol ||f|| (count k = the
    products that contributed to u), else alpha_k = r.z / p.q and
    beta_k = (r.z - 2 alpha_k z.q + alpha_k^2 q.D^-1.q) / r.z.
    In floating point the predicted numerator differs from the explicit one by rounding that
    is amplified where the residual drops sharply; at high contrast the two recurrences then
    follow different (equally valid) finite-precision trajectories. Pinned against pcg() on
    well-conditioned systems (tests/test_oracle_fem.py). Returns as pcg()."""
    f = np.asarray(f, dtype=np.float64)
    fnorm = np.linalg.norm(f)
    if fnorm == 0.0:
        return np.zeros_like(f), 0, True, 0.0
    u = np.zeros_like(f) if x0 is None else np.array(x0, dtype=np.float64)
    r_prev = f - apply_A(u) if np.any(u) else f.copy()
    q_prev = np.zeros_like(f)
    p_prev = np.zeros_like(f)
    alpha = beta = 0.0
    k = 0
    while True:
        r = r_prev - alpha * q_prev
        z = dinv * r
        p = z + beta * p_prev
        u = u + alpha * p_prev
        q = apply_A(p)
        pq, rz, rr, zq, qdq = p @ q, r @ z, r @ r, z @ q, q @ (dinv * q)
        rel = np.sqrt(rr) / fnorm
        if callback is not None:
            callback(k, rel)
        if np.sqrt(rr) <= tol * fnorm:
            return u, k, True, rel
        if k >= max_iters:
            return u, k, False, rel
        if not pq > 0.0:
            raise Breakdown(f"p^T A p = {pq} <= 0 at launch {k} (SPEC:173)")
        alpha_k = rz / pq
        beta = (rz - 2.0 * alpha_k * zq + alpha_k * alpha_k * qdq) / rz
        alpha = alpha_k
        r_prev, q_prev, p_prev = r, q, p
        k += 1
