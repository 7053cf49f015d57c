"""Finite elements: KE, SIMP, assembly, matrix-free apply (oracle; test infrastructure only).

Cites: PAPER:180 ("K(z)u - f = 0, where K and f are the stiffness matrix and the
global force vector"); PAPER:91 (finite element discretisation)
[OP hex8_stiffness] (2x2x2 Gauss quadrature of B^T C B, C isotropic with E = 1);
SPEC:114-122 [OP simp_modulus] E = Emin + z^p (E0 - Emin)
[OP apply_stiffness] (fixed DOFs act as identity rows and columns)
[OP jacobi_diagonal]; SURVEY §8 readings A3, A4, A7.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .grid import CORNERS


def lame(E, nu):
    """Lame parameters of an isotropic solid."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return lam, mu


def elasticity_matrix(E, nu):
    """6x6 isotropic C in Voigt order (xx, yy, zz, xy, yz, zx), engineering shear strains."""
    lam, mu = lame(E, nu)
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    for d in range(3):
        C[d, d] += 2.0 * mu
        C[3 + d, 3 + d] = mu
    return C


def shape_gradients(xi, eta, zeta, h):
    """d N_a / d(x, y, z) at the point (xi, eta, zeta) in [0,1]^3 of a cube of edge h.
    N_a = prod over axes of (x if a_x = 1 else 1 - x)."""
    pt = (xi, eta, zeta)
    dN = np.zeros((3, 8))
    for a, corner in enumerate(CORNERS):
        f = [pt[d] if corner[d] else 1.0 - pt[d] for d in range(3)]
        s = [1.0 if corner[d] else -1.0 for d in range(3)]
        dN[0, a] = s[0] * f[1] * f[2] / h
        dN[1, a] = f[0] * s[1] * f[2] / h
        dN[2, a] = f[0] * f[1] * s[2] / h
    return dN


def strain_displacement(dN):
    """6x24 B with u_e ordered [u_x, u_y, u_z] per corner (SPEC:47 ordering)."""
    B = np.zeros((6, 24))
    for a in range(8):
        x, y, z = dN[0, a], dN[1, a], dN[2, a]
        B[0, 3 * a + 0] = x
        B[1, 3 * a + 1] = y
        B[2, 3 * a + 2] = z
        B[3, 3 * a + 0] = y
        B[3, 3 * a + 1] = x
        B[4, 3 * a + 1] = z
        B[4, 3 * a + 2] = y
        B[5, 3 * a + 0] = z
        B[5, 3 * a + 2] = x
    return B


def element_stiffness(nu, h=1.0, E=1.0):
    """KE = sum over 2x2x2 Gauss points of w |J| B^T C B, unit modulus by default.
    2-point Gauss is exact for the trilinear cube (reading A3)."""
    C = elasticity_matrix(E, nu)
    gp = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))
    w = 0.125 * h ** 3  # weight 1/2 per axis on [0,1], times |J| = h^3
    KE = np.zeros((24, 24))
    for xi in gp:
        for eta in gp:
            for zeta in gp:
                B = strain_displacement(shape_gradients(xi, eta, zeta, h))
                KE += w * B.T @ C @ B
    return KE


def simp(rho, E0, Emin, penal):
    """E = Emin + rho^p (E0 - Emin)  (reading A4)."""
    rho = np.asarray(rho, dtype=np.float64)
    # SPEC:118 requires rho in [0, 1]; reading R3 admits 1e-12 of rounding so that
    # the filtered density P x (row-stochastic P, x in [0, 1]) is accepted.
    if not np.all((rho >= -1e-12) & (rho <= 1.0 + 1e-12)):  # also rejects NaN
        raise ValueError("density outside [0, 1] or NaN (SPEC:118)")
    return Emin + rho ** penal * (E0 - Emin)


def assemble(edof, E, KE, n_dof):
    """Global K = sum_e E_e S_e^T KE S_e as scipy CSR (duplicates summed); no BCs."""
    n_e = edof.shape[0]
    rows = np.repeat(edof, 24, axis=1).ravel()
    cols = np.tile(edof, (1, 24)).ravel()
    vals = (E[:, None] * KE.ravel()[None, :]).ravel()
    K = sp.coo_matrix((vals, (rows, cols)), shape=(n_dof, n_dof)).tocsr()
    K.sum_duplicates()
    assert n_e == E.size
    return K


def apply_bc(K, fixed):
    """K_hat: fixed DOFs become identity rows and columns (reading A7)."""
    free = sp.diags((~fixed).astype(np.float64))
    return (free @ K @ free + sp.diags(fixed.astype(np.float64))).tocsr()


def apply_matfree(u, E, KE, edof, fixed):
    """K_hat u without forming K: element loop (vectorised over elements).
    y = sum_e E_e S_e^T KE S_e (u masked at fixed DOFs); y_i = u_i at fixed DOFs."""
    uu = np.where(fixed, 0.0, u)
    ue = uu[edof]                                  # (N_e, 24)
    ye = (ue @ KE.T) * E[:, None]                  # KE symmetric
    y = np.bincount(edof.ravel(), weights=ye.ravel(), minlength=u.size)
    return np.where(fixed, u, y)


def jacobi_diag(E, KE, edof, fixed):
    """diag(K_hat): sum_e E_e KE_dd over elements touching the DOF; 1 at fixed DOFs."""
    d = np.bincount(edof.ravel(), weights=(E[:, None] * np.diag(KE)[None, :]).ravel(),
                    minlength=fixed.size)
    return np.where(fixed, 1.0, d)
