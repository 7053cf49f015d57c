"""Compliance and its sensitivity (oracle; test infrastructure only).

Cites: Eq. (4) "J(z, u(z)) = f^T u(z)"; Eq. (5)
"g_i = -u^T (dK/dz_i) u"; SPEC:263-271 [OP compliance]
[OP compliance_gradient] (g~_e = -p z~_e^{p-1} (E0 - Emin) u_e^T KE u_e, then
g = P^T g~); SURVEY §8 reading A5 (the (E0 - Emin) factor is kept).
"""
from __future__ import annotations

import numpy as np


def compliance(f, u):
    """c = f^T u  (Eq. 4)."""
    return float(np.dot(f, u))


def element_energy(u, KE, edof, fixed=None):
    """ce_e = u_e^T KE u_e (u masked to 0 at fixed DOFs if a mask is given)."""
    uu = u if fixed is None else np.where(fixed, 0.0, u)
    ue = uu[edof]
    return np.einsum("ei,ij,ej->e", ue, KE, ue)


def sensitivity(rho, u, KE, edof, E0, Emin, penal, fixed=None):
    """dc_e = -u^T (dK/drho_e) u with K = sum_e (Emin + rho_e^p (E0 - Emin)) KE_e (Eq. 5):
    dK/drho_e = p rho_e^{p-1} (E0 - Emin) KE_e, so dc_e = -p rho_e^{p-1} (E0 - Emin) ce_e.
    Returns (dc, ce)."""
    ce = element_energy(u, KE, edof, fixed)
    dc = -penal * rho ** (penal - 1.0) * (E0 - Emin) * ce
    return dc, ce
