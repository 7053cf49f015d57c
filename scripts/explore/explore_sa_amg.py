"""Exploration of SURVEY f2 on the CPU oracle (not a test; calls only oracle/ and inputs):
smoothed-aggregation multigrid with the six rigid-body modes as near-null space, as the
preconditioner of CG, on the cfg3 density recipe at reduced size. Question answered: does a
coarse space that contains the rigid motions of every aggregate (hence of every solid
island held by 1e-9 material) converge in a size-independent number of iterations where
the geometric Galerkin hierarchy of oracle/mg.py does not?

Structured aggregation: 3x3x3 node blocks per level (the coarse "nodes" are the aggregates
on a structured grid, 6 DOFs each); tentative P = per-aggregate orthonormalised rigid modes;
P = (I - omega D^-1 A) P_tent, omega = 4/3 / rho(D^-1 A); A_c = P^T A P; symmetric
block-Jacobi (3x3 or 6x6 diagonal blocks) V-cycle; coarsest exact.
    python scripts/explore/explore_sa_amg.py 4      # 1/4-size cfg3 recipe
"""
import dataclasses
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from oracle.loop import OracleProblem  # noqa: E402
from paper_2104_12282_b200 import inputs  # noqa: E402


def rigid_modes(n3):
    nx, ny, nz = n3
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    x, y, z = (a.ravel().astype(float) for a in (i, j, k))
    o, one = np.zeros_like(x), np.ones_like(x)
    cols = [(one, o, o), (o, one, o), (o, o, one), (-y, x, o), (o, -z, y), (z, o, -x)]
    return np.stack([np.stack(c, axis=1).ravel() for c in cols], axis=1)  # (3 nn, 6)


def aggregates(dims, a=3):
    """Node index -> aggregate index for a structured node grid dims = (mx, my, mz)."""
    mx, my, mz = dims
    gx, gy, gz = -(-mx // a), -(-my // a), -(-mz // a)
    k, j, i = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    agg = (i // a) + gx * ((j // a) + gy * (k // a))
    return agg.ravel(), (gx, gy, gz)


def strength_aggregates(A, bs, theta=0.08):
    """Greedy standard aggregation on the node graph of strong connections: i-j strong if
    ||A_ij||_F >= theta sqrt(||A_ii||_F ||A_jj||_F) (block norms). Phase 1: every node whose
    strong neighbourhood is free seeds an aggregate of it; phase 2: leftovers join the
    aggregate of a strong neighbour; phase 3: the rest form aggregates of themselves."""
    A = sp.csr_matrix(A)
    n = A.shape[0] // bs
    Ab = sp.bsr_matrix(A, blocksize=(bs, bs))
    Ab.sort_indices()
    norms = np.sqrt((Ab.data ** 2).sum(axis=(1, 2)))
    rows = np.repeat(np.arange(n), np.diff(Ab.indptr))
    cols = Ab.indices
    diag = np.zeros(n)
    dm = rows == cols
    diag[rows[dm]] = norms[dm]
    strong = (norms >= theta * np.sqrt(diag[rows] * diag[cols])) & ~dm
    S = sp.csr_matrix((np.ones(strong.sum()), (rows[strong], cols[strong])), shape=(n, n))
    indptr, ind = S.indptr, S.indices
    agg = -np.ones(n, dtype=np.int64)
    na = 0
    for i in range(n):  # phase 1
        nb = ind[indptr[i]:indptr[i + 1]]
        if agg[i] < 0 and (agg[nb] < 0).all():
            agg[i] = na
            agg[nb] = na
            na += 1
    for i in np.nonzero(agg < 0)[0]:  # phase 2
        nb = ind[indptr[i]:indptr[i + 1]]
        got = agg[nb][agg[nb] >= 0]
        if got.size:
            agg[i] = got[0]
    for i in np.nonzero(agg < 0)[0]:  # phase 3
        agg[i] = na
        na += 1
    return agg, na


def tentative(B, agg, nagg, bs):
    """Block-diagonal P_tent with orthonormal columns spanning B on every aggregate; returns
    (P_tent, B_coarse) with B = P_tent B_coarse (bs DOFs per fine node, 6 near-null vectors)."""
    nn = B.shape[0] // bs
    rows, cols, vals = [], [], []
    Bc = np.zeros((6 * nagg, 6))
    dof_agg = np.repeat(agg, bs)
    order = np.argsort(dof_agg, kind="stable")
    bounds = np.searchsorted(dof_agg[order], np.arange(nagg + 1))
    for g in range(nagg):
        idx = order[bounds[g]:bounds[g + 1]]
        # rank-revealing factorisation B_agg = Q R (aggregates with fewer than 6 DOFs or
        # with fixed nodes have rank < 6: the missing columns of Q are zero)
        U, sv, Vt = np.linalg.svd(B[idx], full_matrices=False)
        r = int((sv > 1e-12 * max(sv.max(), 1e-300)).sum()) if sv.size else 0
        Q = np.zeros((len(idx), 6))
        R = np.zeros((6, 6))
        Q[:, :r] = U[:, :r]
        R[:r] = sv[:r, None] * Vt[:r]
        rows.append(np.repeat(idx, 6)); cols.append(np.tile(6 * g + np.arange(6), len(idx)))
        vals.append(Q.ravel())
        Bc[6 * g:6 * g + 6] = R
    P = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(bs * nn, 6 * nagg))
    return P, Bc


def block_dinv(A, bs):
    A = sp.csr_matrix(A)
    n = A.shape[0] // bs
    D = np.zeros((n, bs, bs))
    for a in range(bs):
        for b in range(bs):
            D[:, a, b] = A[a::bs, b::bs].diagonal()
    return np.linalg.inv(D)


def apply_bd(Dinv, r, bs):
    return np.einsum("nab,nb->na", Dinv, r.reshape(-1, bs)).ravel()


def spectral_radius(A, Dinv, bs, its=30):
    v = np.random.default_rng(0).standard_normal(A.shape[0])
    lam = 0.0
    for _ in range(its):
        w = apply_bd(Dinv, A @ v, bs)
        lam = np.linalg.norm(w) / np.linalg.norm(v)
        v = w / np.linalg.norm(w)
    return lam


def hierarchy(A, fixed, n3, max_coarse=600, strength=False):
    levels = []
    B = rigid_modes(n3)
    B[fixed] = 0.0
    dims = tuple(n + 1 for n in n3)
    bs = 3
    while True:
        Dinv = block_dinv(A, bs)
        levels.append({"A": A, "Dinv": Dinv, "bs": bs})
        if A.shape[0] <= max_coarse or (not strength and max(dims) <= 2):
            break
        if strength:
            agg, nagg = strength_aggregates(A, bs, theta=0.08 if bs == 3 else 0.0)
            cdims = (nagg, 1, 1)
            print(f"  level {len(levels) - 1}: {A.shape[0] // bs} nodes -> {nagg} aggregates", flush=True)
            if nagg > 0.5 * (A.shape[0] // bs):  # aggregation stalled: stop coarsening here
                break
        else:
            agg, cdims = aggregates(dims)
            nagg = int(np.prod(cdims))
        Pt, Bc = tentative(B, agg, nagg, bs)
        rho = spectral_radius(A, Dinv, bs)
        S = sp.csr_matrix(A)
        # P = (I - omega D^-1 A) P_tent
        nb = Dinv.shape[0]
        Dblk = sp.bsr_matrix((Dinv, np.arange(nb), np.arange(nb + 1)), shape=(bs * nb, bs * nb)).tocsr()
        P = (Pt - (4.0 / 3.0 / rho) * (Dblk @ (S @ Pt))).tocsr()
        levels[-1]["P"] = P
        A = (P.T @ S @ P).tocsr()
        # drop numerically empty coarse DOFs (aggregates of fixed nodes only)
        d = A.diagonal()
        keep = d > 1e-14 * d.max()
        if not keep.all():
            A = A + sp.diags((~keep).astype(float))
        B, dims, bs = Bc, cdims, 6
    return levels


def vcycle(levels, l, b, nu=2, omega=0.6, cache=None):
    L = levels[l]
    A, Dinv, bs = L["A"], L["Dinv"], L["bs"]
    if l == len(levels) - 1:
        if "lu" not in cache:
            cache["lu"] = spla.splu(sp.csc_matrix(A))
        return cache["lu"].solve(b)
    x = np.zeros_like(b)
    for _ in range(nu):
        x = x + omega * apply_bd(Dinv, b - A @ x, bs)
    P = L["P"]
    x = x + P @ vcycle(levels, l + 1, P.T @ (b - A @ x), nu, omega, cache)
    for _ in range(nu):
        x = x + omega * apply_bd(Dinv, b - A @ x, bs)
    return x


def pcg(levels, f, tol=1e-10, max_iters=3000, nu=2, omega=0.6):
    A = levels[0]["A"]
    cache = {}
    u = np.zeros_like(f)
    r = f.copy()
    z = vcycle(levels, 0, r, nu, omega, cache)
    p = z.copy()
    rz = r @ z
    fn = np.linalg.norm(f)
    for k in range(1, max_iters + 1):
        q = A @ p
        al = rz / (p @ q)
        u += al * p
        r -= al * q
        if np.linalg.norm(r) <= tol * fn:
            return u, k
        z = vcycle(levels, 0, r, nu, omega, cache)
        rzn = r @ z
        p = z + (rzn / rz) * p
        rz = rzn
    return u, max_iters


if __name__ == "__main__":
    s = int(sys.argv[1]) if len(sys.argv) > 1 else 4  # [--strength]
    p = dataclasses.replace(inputs.CONFIGS["cfg3"], nx=224 // s, ny=112 // s, nz=56 // s)
    rho = inputs.density_blobs_beta(p, sigma=6.0 / s)
    op = OracleProblem(p)
    A = op.Khat(rho)
    t0 = time.time()
    strength = "--strength" in sys.argv
    levels = hierarchy(A, op.fixed, (p.nx, p.ny, p.nz), strength=strength)
    print("levels", [L["A"].shape[0] for L in levels], f"setup {time.time() - t0:.1f}s", flush=True)
    for nu, om in [(2, 0.6), (2, 0.4)]:
        t0 = time.time()
        u, k = pcg(levels, op.f, nu=nu, omega=om)
        tag = "strength" if strength else "structured"
        print(f"cfg3/{s} SA-AMG ({tag}) nu={nu} omega={om}: {k} iterations, {time.time() - t0:.1f}s", flush=True)
