"""Galerkin multigrid hierarchy and MG-preconditioned CG (oracle; test infrastructure only).

SURVEY §8 f2 ("Multigrid-preconditioned CG (geometric, on the structured grid)")
and PAPER:184 ("Iterative solvers such as preconditioned conjugate gradient (PCG) and
multi-grid methods are typically used"). The paper names the method but fixes none of its
parts, so the choices below are this build's readings (reading R5):

* Coarse nodes per axis (n fine elements along the axis, n >= 2): fine positions
  0, 2, 4, ..., and the last position is n; if n is odd the last coarse interval spans 3
  fine elements (positions ..., n-3, n). Axes with n <= 1 are not coarsened.
* P: linear interpolation per axis, tensor product over the axes, identity over the 3
  displacement components. Masked: P_m = diag(free_f) P diag(free_c).
* A coarse DOF is fixed iff the fine DOF at the coincident position is fixed.
* Galerkin coarse operator A_c = P_m^T A_f P_m + diag(fixed_c) (identity rows/columns at
  fixed DOFs, as K_hat, reading A7).
* V-cycle: nu sweeps of damped block Jacobi (3x3 diagonal blocks, weight omega) before and
  after the coarse correction; the coarsest level solved exactly.
* Outer iteration: CG preconditioned by one V-cycle from zero (symmetric: the same sweeps
  before and after, R = P^T), x0 = 0, stop on ||r_k|| <= tol ||f|| (reading A11).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def coarse_positions(n: int) -> np.ndarray:
    """Fine node positions of the coarse nodes along an axis of n elements."""
    if n <= 1:
        return np.arange(n + 1)
    m = n // 2 + 1
    pos = 2 * np.arange(m)
    pos[-1] = n
    return pos


def prolong_1d(n: int) -> sp.csr_matrix:
    """(n+1) x m linear interpolation from the coarse positions to every fine node."""
    pos = coarse_positions(n)
    rows, cols, vals = [], [], []
    for I in range(len(pos)):
        rows.append(pos[I]); cols.append(I); vals.append(1.0)
        if I + 1 < len(pos):
            a, b = pos[I], pos[I + 1]
            for i in range(a + 1, b):
                rows += [i, i]
                cols += [I, I + 1]
                vals += [(b - i) / (b - a), (i - a) / (b - a)]
    return sp.csr_matrix((vals, (rows, cols)), shape=(n + 1, len(pos)))


def prolongation(n3) -> sp.csr_matrix:
    """DOF prolongation for a grid of n3 = (nx, ny, nz) elements (node order x fastest,
    DOF = 3 node + component)."""
    nx, ny, nz = n3
    P = sp.kron(prolong_1d(nz), sp.kron(prolong_1d(ny), sp.kron(prolong_1d(nx), sp.identity(3))))
    return sp.csr_matrix(P)


def coarse_elems(n3):
    return tuple(len(coarse_positions(n)) - 1 for n in n3)


def coarse_fixed(fixed_f: np.ndarray, n3) -> np.ndarray:
    """Coarse DOF fixed iff the fine DOF at the coincident node is fixed."""
    nx, ny, nz = n3
    px, py, pz = (coarse_positions(n) for n in n3)
    K, J, I = np.meshgrid(pz, py, px, indexing="ij")
    fine_node = (I + (nx + 1) * (J + (ny + 1) * K)).ravel()
    ff = fixed_f.reshape(-1, 3)
    return ff[fine_node].ravel().copy()


def galerkin(A_f: sp.spmatrix, n3, fixed_f: np.ndarray):
    """(A_c, P_m, fixed_c) with A_c = P_m^T A_f P_m + diag(fixed_c)."""
    fixed_c = coarse_fixed(fixed_f, n3)
    P = prolongation(n3)
    Pm = sp.diags((~fixed_f).astype(np.float64)) @ P @ sp.diags((~fixed_c).astype(np.float64))
    Pm = sp.csr_matrix(Pm)
    A_c = (Pm.T @ A_f @ Pm + sp.diags(fixed_c.astype(np.float64))).tocsr()
    return A_c, Pm, fixed_c


def hierarchy(A0: sp.spmatrix, n3, fixed0: np.ndarray, max_coarse_dofs: int = 400):
    """Levels [(A_l, n3_l, fixed_l, P_l)] where P_l maps level l+1 to level l."""
    levels = [{"A": sp.csr_matrix(A0), "n3": tuple(n3), "fixed": fixed0, "P": None}]
    while levels[-1]["A"].shape[0] > max_coarse_dofs and max(levels[-1]["n3"]) > 1:
        L = levels[-1]
        A_c, Pm, fixed_c = galerkin(L["A"], L["n3"], L["fixed"])
        L["P"] = Pm
        levels.append({"A": A_c, "n3": coarse_elems(L["n3"]), "fixed": fixed_c, "P": None})
    return levels


def block_diag_inverse(A: sp.spmatrix) -> np.ndarray:
    """Inverses of the 3x3 diagonal blocks of A, shape (n_node, 3, 3)."""
    A = sp.csr_matrix(A)
    n = A.shape[0] // 3
    D = np.zeros((n, 3, 3))
    for a in range(3):
        for b in range(3):
            D[:, a, b] = A[a::3, b::3].diagonal()
    return np.linalg.inv(D)


def vcycle(levels, l: int, b: np.ndarray, nu: int, omega: float, cache: dict) -> np.ndarray:
    """One V-cycle on level l from x = 0 (block Jacobi, nu sweeps each side)."""
    L = levels[l]
    A = L["A"]
    if l == len(levels) - 1:
        if "lu" not in cache:
            cache["lu"] = spla.splu(sp.csc_matrix(A))
        return cache["lu"].solve(b)
    key = ("Dinv", l)
    if key not in cache:
        cache[key] = block_diag_inverse(A)
    Dinv = cache[key]

    def smooth(x):
        r = (b - A @ x).reshape(-1, 3)
        return x + omega * np.einsum("nab,nb->na", Dinv, r).ravel()

    x = np.zeros_like(b)
    for _ in range(nu):
        x = smooth(x)
    r = b - A @ x
    P = L["P"]
    x = x + P @ vcycle(levels, l + 1, P.T @ r, nu, omega, cache)
    for _ in range(nu):
        x = smooth(x)
    return x


def mgpcg(levels, f: np.ndarray, tol: float = 1e-10, max_iters: int = 1000, nu: int = 2,
          omega: float = 0.6):
    """CG preconditioned by one V-cycle; returns (u, iterations, ||r||/||f||)."""
    A = levels[0]["A"]
    cache: dict = {}
    u = np.zeros_like(f)
    r = f.copy()
    fn = np.linalg.norm(f)
    z = vcycle(levels, 0, r, nu, omega, cache)
    p = z.copy()
    rz = r @ z
    for k in range(1, max_iters + 1):
        q = A @ p
        alpha = rz / (p @ q)
        u += alpha * p
        r -= alpha * q
        if np.linalg.norm(r) <= tol * fn:
            return u, k, np.linalg.norm(r) / fn
        z = vcycle(levels, 0, r, nu, omega, cache)
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return u, max_iters, np.linalg.norm(r) / fn
