"""Density filter P (oracle; test infrastructure only).

Cites: Eq. (4) "V(z) = v^T P z - V_max", PAPER:180 ("P is the density
filter matrix"), PAPER:184 ("dV/dz = P^T v"); SPEC:217-225 [OP build_filter]:
w~_ij = max(0, R - ||c_i - c_j||_2) over element centroids, rows normalised to
sum 1; SPEC:226-238 [OP apply / apply_transpose]; SURVEY reading A15 (tap set:
integer offsets d with rmin - sqrt(dx^2 + dy^2 + dz^2) > 0 in fp64, boundary
truncated, no padding) and A16 (v = 1 per element, dv = P^T 1).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def taps(rmin):
    """[(dx, dy, dz, w)] for all integer offsets with w = rmin - |d| > 0, order dz, dy, dx ascending."""
    r = int(np.ceil(rmin))
    out = []
    for dz in range(-r, r + 1):
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                w = rmin - np.sqrt(float(dx * dx + dy * dy + dz * dz))
                if w > 0.0:
                    out.append((dx, dy, dz, w))
    return out


def filter_matrices(nx, ny, nz, rmin):
    """(H, Hs): H_ij = max(0, rmin - dist(c_i, c_j)) as CSR, Hs_i = sum_j H_ij."""
    n_e = nx * ny * nz
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    e = i + nx * (j + ny * k)
    rows, cols, vals = [], [], []
    for dx, dy, dz, w in taps(rmin):
        ii, jj, kk = i + dx, j + dy, k + dz
        ok = (ii >= 0) & (ii < nx) & (jj >= 0) & (jj < ny) & (kk >= 0) & (kk < nz)
        rows.append(e[ok])
        cols.append((ii + nx * (jj + ny * kk))[ok])
        vals.append(np.full(int(ok.sum()), w))
    H = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n_e, n_e))
    Hs = np.asarray(H.sum(axis=1)).ravel()
    return H, Hs


def filter_matrix(nx, ny, nz, rmin):
    """P = diag(1/Hs) H  (row-stochastic)."""
    H, Hs = filter_matrices(nx, ny, nz, rmin)
    return (sp.diags(1.0 / Hs) @ H).tocsr()


def apply(P, x):
    """Forward filter rho~ = P x."""
    return P @ x


def apply_transpose(P, v):
    """P^T v, literally (chain rule of the density filter; the 'filtered dc' of BASELINE.json)."""
    return P.T @ v


def volume_gradient(P):
    """dV/dz = P^T v with v = 1 (reading A16)."""
    return P.T @ np.ones(P.shape[0])


def neighbor_counts(nx, ny, nz, rmin):
    """Number of in-domain taps per element (integer; for bit-exact parity)."""
    H, _ = filter_matrices(nx, ny, nz, rmin)
    return np.diff(H.indptr).astype(np.int64)


def hs_of(nx, ny, nz, rmin, elems):
    """Hs_e = sum of the in-domain tap weights of element e, for the listed elements only
    (same tap set and summation order as filter_matrices; for grids whose full H does not fit
    in memory - the paper's 1551-tap radius on its 1.46M-element Mesh 3)."""
    e = np.asarray(elems, dtype=np.int64)
    i, j, k = e % nx, (e // nx) % ny, e // (nx * ny)
    out = np.zeros(e.size)
    for dx, dy, dz, w in taps(rmin):  # tap by tap, vectorised over the elements
        ok = (i + dx >= 0) & (i + dx < nx) & (j + dy >= 0) & (j + dy < ny) & (k + dz >= 0) & (k + dz < nz)
        out += np.where(ok, w, 0.0)
    return out


def filter_rows(nx, ny, nz, rmin, elems, x, transpose=False):
    """(P x)_e or (P^T x)_e for the listed elements only, by the definitions of SPEC:220-233:
    (P x)_e = sum_j w_ej x_j / Hs_e; (P^T v)_e = sum_i w_ie v_i / Hs_i over the in-domain taps
    (w symmetric). Element by element (sampled parity at sizes where P cannot be formed)."""
    t = taps(rmin)
    out = np.empty(len(elems))
    for q, e in enumerate(np.asarray(elems).tolist()):
        i, j, k = e % nx, (e // nx) % ny, e // (nx * ny)
        nb, wt = [], []
        for dx, dy, dz, w in t:
            if 0 <= i + dx < nx and 0 <= j + dy < ny and 0 <= k + dz < nz:
                nb.append((i + dx) + nx * ((j + dy) + ny * (k + dz)))
                wt.append(w)
        nb, wt = np.array(nb), np.array(wt)
        if transpose:
            out[q] = float(np.sum(wt * x[nb] / hs_of(nx, ny, nz, rmin, nb)))
        else:
            out[q] = float(np.sum(wt * x[nb])) / hs_of(nx, ny, nz, rmin, [e])[0]
    return out
