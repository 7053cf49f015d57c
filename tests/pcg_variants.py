"""CPU models of PCG recurrences for iteration-count pins (test infrastructure; not the
oracle, which is the textbook method of oracle/solve.py).

single_pass_pcg follows the recurrence the fused CUDA kernel implements (DESIGN.md §5.3,
reading R1), written independently of the CUDA code from that description: launch k forms
    r_k = r_{k-1} - alpha_{k-1} q_{k-1},  z_k = D^-1 r_k,  p_k = z_k + beta_{k-1} p_{k-1},
    u_k = u_{k-1} + alpha_{k-1} p_{k-1},  q_k = K p_k,
reduces p.q, r.z, r.r, z.q and q.D^-1.q, stops when ||r_k|| <= tol ||f||, else sets
    alpha_k = (r.z)/(p.q),  beta_k = (r.z - 2 alpha_k z.q + alpha_k^2 q.D^-1.q) / (r.z)
(the predicted r_{k+1}.z_{k+1} over the explicit r_k.z_k). The count is the index k of the
launch that met the tolerance (= the number of K p products that contributed to u)."""
from __future__ import annotations

import numpy as np


def single_pass_pcg(apply_A, dinv, f, tol=1e-10, max_iters=100000, callback=None):
    fnorm = np.linalg.norm(f)
    u = np.zeros_like(f)
    r_prev = f.copy()           # r_{-1} = f - K u0 with u0 = 0
    q_prev = np.zeros_like(f)   # q_{-1} = 0
    p_prev = np.zeros_like(f)   # p_{-1} = 0
    alpha = beta = 0.0
    k = 0
    while True:
        r = r_prev - alpha * q_prev
        z = dinv * r
        p = z + beta * p_prev
        u += alpha * p_prev
        q = apply_A(p)
        pq, rz, rr = p @ q, r @ z, r @ r
        zq, qdq = z @ q, q @ (dinv * q)
        rel = np.sqrt(rr) / fnorm
        if callback is not None:
            callback(k, rel)
        if np.sqrt(rr) <= tol * fnorm:
            return u, k, True, rel
        if k >= max_iters:
            return u, k, False, rel
        if not pq > 0.0:
            raise RuntimeError("breakdown")
        alpha_k = rz / pq
        rz_next = rz - 2.0 * alpha_k * zq + alpha_k * alpha_k * qdq
        beta = rz_next / rz
        alpha = alpha_k
        r_prev, q_prev, p_prev = r, q, p
        k += 1
