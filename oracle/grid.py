"""Structured hexahedral grid, numbering and boundary conditions (oracle; test infrastructure only).

Cites: SPEC:22-31 [TYPE StructuredGrid] (x fastest, then y, then z; 24 DOFs per
element), SPEC:44-52 [OP element_dofs], PAPER:180 ("K(z)u - f = 0", f is the
global force vector), PAPER:207 (cantilever: fixed face x=0, distributed load;
MBB), BASELINE.json configs[0..4] and SURVEY.md §8(c2) readings A1, A8-A10.
"""
from __future__ import annotations

import numpy as np

# Corner order of the 8-node element: local (ax, ay, az).
CORNERS = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
           (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def counts(nx, ny, nz):
    """(N_e, N_n, N_dof): SPEC:29 node count (nx+1)(ny+1)(nz+1), N_s = 3 * nodes."""
    n_e = nx * ny * nz
    n_n = (nx + 1) * (ny + 1) * (nz + 1)
    return n_e, n_n, 3 * n_n


def node_id(i, j, k, nx, ny):
    """Node (i,j,k) -> n = i + (nx+1)(j + (ny+1)k)  (x fastest)."""
    return i + (nx + 1) * (j + (ny + 1) * k)


def element_id(i, j, k, nx, ny):
    """Element (i,j,k) -> e = i + nx(j + ny k)."""
    return i + nx * (j + ny * k)


def element_dofs(nx, ny, nz):
    """(N_e, 24) int64: row e lists DOFs 3*n_a + c for corners a in CORNERS, c = x, y, z."""
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    out = np.empty((i.size, 24), dtype=np.int64)
    for a, (ax, ay, az) in enumerate(CORNERS):
        n = node_id(i + ax, j + ay, k + az, nx, ny)
        for c in range(3):
            out[:, 3 * a + c] = 3 * n + c
    return out


def _nodes_where(nx, ny, nz, pred):
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    m = pred(i, j, k)
    return node_id(i[m], j[m], k[m], nx, ny)


def cantilever_bc(nx, ny, nz, load_total=-1.0):
    """Cantilever ("fixed on its face x=0 and subjected to a distributed load";
    BASELINE.json configs[0]: "x=0 face fully clamped; total load -1 in z spread evenly
    over the nodes of the bottom edge of the x=max face").

    Returns (fixed_mask[N_dof] bool, load_dofs int64, load_vals float64).
    Reading A8: equal weights load_total/(ny+1) on nodes (nx, j, 0), j = 0..ny.
    """
    _, _, n_dof = counts(nx, ny, nz)
    fixed = np.zeros(n_dof, dtype=bool)
    for n in _nodes_where(nx, ny, nz, lambda i, j, k: i == 0):
        fixed[3 * n: 3 * n + 3] = True
    nodes = np.array([node_id(nx, j, 0, nx, ny) for j in range(ny + 1)], dtype=np.int64)
    dofs = 3 * nodes + 2
    vals = np.full(dofs.size, load_total / (ny + 1))
    return fixed, dofs, vals


def mbb_half_bc(nx, ny, nz, load_total=-1.0):
    """MBB half-beam (BASELINE.json configs[2]): symmetry u_x = 0 on the x=0 face; roller
    u_z = 0 on the bottom edge line (nx, j, 0); unit -z line load on the top edge at x=0.
    Reading A9: u_y = 0 at node (nx, 0, 0) removes the free y-translation.
    Reading A10: total load_total with equal weights over nodes (0, j, nz)."""
    _, _, n_dof = counts(nx, ny, nz)
    fixed = np.zeros(n_dof, dtype=bool)
    for n in _nodes_where(nx, ny, nz, lambda i, j, k: i == 0):
        fixed[3 * n + 0] = True
    for j in range(ny + 1):
        fixed[3 * node_id(nx, j, 0, nx, ny) + 2] = True
    fixed[3 * node_id(nx, 0, 0, nx, ny) + 1] = True
    nodes = np.array([node_id(0, j, nz, nx, ny) for j in range(ny + 1)], dtype=np.int64)
    dofs = 3 * nodes + 2
    vals = np.full(dofs.size, load_total / (ny + 1))
    return fixed, dofs, vals


def bc_for(kind, nx, ny, nz, load_total=-1.0):
    if kind == 1:
        return cantilever_bc(nx, ny, nz, load_total)
    if kind == 2:
        return mbb_half_bc(nx, ny, nz, load_total)
    raise ValueError(f"unknown BC kind {kind}")


def load_vector(n_dof, load_dofs, load_vals):
    f = np.zeros(n_dof)
    np.add.at(f, load_dofs, load_vals)
    return f
