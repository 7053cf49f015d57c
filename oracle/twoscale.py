"""Two-scale coarse path (oracle; test infrastructure only).

Cites: PAPER:150-157 §"Two-scale Optimization" ("we segment the design variables z into
small subsets ... coarse-grained design variable vector z_C so that each of its component
is the averaged value of z in each subset"); PAPER:184-186 ("3D blocks of uniform
dimensions N_B x N_B x N_B ... K_C(z_C) u_C - f_C = 0"); Alg. 1 lines 3-4;
SPEC:364-391 [OP coarsen_density], [OP restrict_bc], [OP solve_coarse].

Reading R4: the "nearest coarse node" of fine node index i along an axis is
I = floor(i / N_B + 1/2) (ties go to the larger index); a coarse DOF is fixed iff any fine
node whose nearest coarse node it is has that DOF fixed; fine loads are summed onto the
nearest coarse node of their DOF; the coarse element edge is N_B h.
"""
from __future__ import annotations

import numpy as np

from . import grid


def coarsen(z, nx, ny, nz, nb):
    """z_C[b] = mean of z over block b of nb^3 elements; z in element order
    e = i + nx (j + ny k). Blocks in the same order on the coarse grid."""
    if nx % nb or ny % nb or nz % nb:
        raise ValueError("block size must divide the grid (SPEC:386)")
    a = np.asarray(z, dtype=np.float64).reshape(nz // nb, nb, ny // nb, nb, nx // nb, nb)
    return a.mean(axis=(1, 3, 5)).ravel()


def nearest(i, nb):
    """Nearest coarse index of fine index i (reading R4: ties go up)."""
    return (2 * np.asarray(i) + nb) // (2 * nb)


def restrict_bc(nx, ny, nz, nb, fixed, load_dofs, load_vals):
    """SPEC:374-382 restrict_bc: (fixed_C[N_dof_C] bool, load_dofs_C, load_vals_C)."""
    cx, cy, cz = nx // nb, ny // nb, nz // nb
    _, n_n, _ = grid.counts(nx, ny, nz)
    _, _, n_dof_c = grid.counts(cx, cy, cz)
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    I, J, K = nearest(i.ravel(), nb), nearest(j.ravel(), nb), nearest(k.ravel(), nb)
    cnode = I + (cx + 1) * (J + (cy + 1) * K)      # fine node -> nearest coarse node
    fixed = np.asarray(fixed, dtype=bool).reshape(n_n, 3)
    fixed_c = np.zeros((n_dof_c // 3, 3), dtype=bool)
    for c in range(3):
        np.logical_or.at(fixed_c[:, c], cnode[fixed[:, c]], True)
    f_c = np.zeros(n_dof_c)
    ld = np.asarray(load_dofs, dtype=np.int64)
    np.add.at(f_c, 3 * cnode[ld // 3] + ld % 3, np.asarray(load_vals, dtype=np.float64))
    dofs_c = np.flatnonzero(f_c)
    return fixed_c.ravel(), dofs_c, f_c[dofs_c]
