"""Pins of the oracle's compliance / sensitivity / filter / OC against finite differences,
identities, closed forms and brute force (not against itself).  CPU only."""
import math

import numpy as np
import pytest

from oracle import fem, filt, oc, sens
from oracle.loop import OracleProblem, simp_loop
from paper_2104_12282_b200 import inputs


# ------------------------------------------------------------------ compliance / sensitivity
def _fd_problem():
    p = inputs.Problem("fd", 4, 2, 2)
    rho = np.random.default_rng(5).uniform(0.3, 0.9, p.n_elem)
    return p, OracleProblem(p), rho


def test_compliance_energy_identity():
    # SPEC:271, SURVEY A-6: f^T u = u^T K_hat u at the solution
    p, op, rho = _fd_problem()
    u = op.solve_direct(rho)
    assert math.isclose(op.compliance(u), u @ op.apply(rho, u), rel_tol=1e-12)
    E = op.E(rho)
    _, ce = op.sensitivity(rho, u)
    assert math.isclose(op.compliance(u), float(E @ ce), rel_tol=1e-12)
    # SPEC:269-270 trivial cases
    assert sens.compliance(op.f, np.zeros(op.n_dof)) == 0.0


def test_sensitivity_finite_difference():
    """Eq. (5) vs central differences of J(rho) = f^T u(rho), step 1e-6, direct solves."""
    p, op, rho = _fd_problem()
    u = op.solve_direct(rho)
    dc, _ = op.sensitivity(rho, u)
    h = 1e-6
    for e in range(p.n_elem):
        rp = rho.copy(); rp[e] += h
        rm = rho.copy(); rm[e] -= h
        fd = (op.compliance(op.solve_direct(rp)) - op.compliance(op.solve_direct(rm))) / (2 * h)
        assert abs(fd - dc[e]) <= 1e-6 * abs(dc[e]), (e, fd, dc[e])
    assert (dc <= 0).all()


def test_sensitivity_general_adjoint_path():
    """Eq. (3) with an explicit adjoint solve reduces to Eq. (5)."""
    p, op, rho = _fd_problem()
    Kh = op.Khat(rho).toarray()
    u = np.linalg.solve(Kh, op.f)
    adj = np.linalg.solve(Kh.T, op.f)  # (dr/du)^-T dJ/du with J = f^T u, r = K u - f
    g = np.zeros(p.n_elem)
    free = ~op.fixed
    for e in range(p.n_elem):
        dK = np.zeros_like(Kh)
        d = op.edof[e]
        dK[np.ix_(d, d)] = p.penal * rho[e] ** (p.penal - 1) * (p.E0 - p.Emin) * op.KE
        dK[~free, :] = 0.0
        dK[:, ~free] = 0.0
        g[e] = 0.0 - adj @ (dK @ u)  # dJ/dz = 0 explicitly
    dc, _ = op.sensitivity(rho, u)
    assert np.allclose(g, dc, rtol=1e-9, atol=0)


def test_homogeneity_and_load_scaling():
    """SURVEY A-5: sum_e rho_e dc_e = -p (c - Emin sum_e ce_e); f -> a f scales dc by a^2."""
    p, op, rho = _fd_problem()
    u = op.solve_direct(rho)
    c = op.compliance(u)
    dc, ce = op.sensitivity(rho, u)
    lhs = rho @ dc
    rhs = -p.penal * (c - p.Emin * ce.sum())
    assert math.isclose(lhs, rhs, rel_tol=1e-11)
    dc2, _ = op.sensitivity(rho, 3.0 * u)
    assert np.allclose(dc2, 9.0 * dc, rtol=1e-13)
    z, _ = op.sensitivity(rho, np.zeros(op.n_dof))
    assert not z.any()


# ------------------------------------------------------------------ filter
@pytest.mark.parametrize("rmin,ntaps,interior,corner", [
    (1.5, 19, 22.5 - 12 * math.sqrt(2), 3.2573593128807152),
    (2.0, 27, 48 - 12 * math.sqrt(2) - 8 * math.sqrt(3), 7.025308505311838),
    (3.0, 93, 261 - 36 * math.sqrt(2) - 8 * math.sqrt(3) - 24 * math.sqrt(5) - 24 * math.sqrt(6),
     24.775150037724988),
])
def test_filter_closed_forms(rmin, ntaps, interior, corner):
    # SURVEY App. A-9; interior Hs written as a closed form over tap shells
    assert len(filt.taps(rmin)) == ntaps
    H, Hs = filt.filter_matrices(9, 9, 9, rmin)
    assert math.isclose(Hs[4 + 9 * (4 + 9 * 4)], interior, rel_tol=1e-13)
    assert math.isclose(Hs[0], corner, rel_tol=1e-13)
    nc = filt.neighbor_counts(9, 9, 9, rmin)
    assert nc[4 + 9 * (4 + 9 * 4)] == ntaps


def test_filter_properties():
    nx, ny, nz = 7, 4, 5
    for rmin in (0.9, 1.5, 2.0, 3.0):
        P = filt.filter_matrix(nx, ny, nz, rmin)
        n = nx * ny * nz
        assert np.allclose(P @ np.ones(n), 1.0, rtol=0, atol=1e-14)  # SPEC:212 rows sum 1
        rng = np.random.default_rng(1)
        v, z = rng.standard_normal(n), rng.uniform(0, 1, n)
        assert math.isclose(filt.apply_transpose(P, v) @ z, v @ filt.apply(P, z), rel_tol=1e-12)
        assert np.allclose(filt.apply(P, np.full(n, 0.37)), 0.37, rtol=1e-14)
        pz = filt.apply(P, z)
        assert pz.min() >= z.min() - 1e-15 and pz.max() <= z.max() + 1e-15  # convex combination
        if rmin < 1.0:
            assert (P != __import__("scipy.sparse", fromlist=["eye"]).eye(n)).nnz == 0
    # (3,1,1), R = 1.5, middle row weights proportional to (0.5, 1.5, 0.5)
    P = filt.filter_matrix(3, 1, 1, 1.5).toarray()
    assert np.allclose(P[1], np.array([0.5, 1.5, 0.5]) / 2.5, rtol=1e-15)


# ------------------------------------------------------------------ OC
def _oc_case(seed, n=(6, 4, 3), rmin=1.5, volfrac=0.3):
    nx, ny, nz = n
    P = filt.filter_matrix(nx, ny, nz, rmin)
    rng = np.random.default_rng(seed)
    ne = nx * ny * nz
    x = rng.uniform(0.05, 0.95, ne)
    g = -rng.uniform(0.01, 10.0, ne) * 10.0 ** rng.uniform(-3, 3, ne)
    dv = filt.volume_gradient(P)
    return x, g, dv, P, volfrac


@pytest.mark.parametrize("seed", range(40))
def test_oc_invariants(seed):
    """box, move limits, volume feasibility, V(lambda) monotone (A17)."""
    x, g, dv, P, vf = _oc_case(seed, volfrac=0.2 + 0.02 * (seed % 10))
    xn, lam, steps, trace = oc.oc_update(x, g, dv, P, vf, 0.2, 0.5)
    assert (xn >= 0).all() and (xn <= 1).all()
    assert (np.abs(xn - x) <= 0.2 + 1e-15).all()
    target = vf * x.size
    if steps > 0:
        assert 50 <= steps <= 64
        assert np.sum(P @ xn) <= target * (1 + 1e-12)
        # just below lambda the volume exceeds the target (bracket is tight)
        xl = oc.x_new(x, g, dv, lam * (1 - 1e-12), 0.2, 0.5)
        assert np.sum(P @ xl) >= np.sum(P @ xn)
        assert abs(np.sum(P @ xn) - target) <= 1e-9 * target
    lams = np.geomspace(1e-6, 1e6, 50)
    vols = [np.sum(P @ oc.x_new(x, g, dv, l, 0.2, 0.5)) for l in lams]
    assert all(a >= b - 1e-12 for a, b in zip(vols, vols[1:]))  # SPEC:331 monotone


def test_oc_uniform_case():
    # uniform g, dv, x -> uniform volume-feasible x_new with equality
    n = 5 * 4 * 3
    P = filt.filter_matrix(5, 4, 3, 1.0)  # identity filter -> dv = 1 uniform
    x = np.full(n, 0.35)
    g = np.full(n, -2.0)
    xn, lam, steps, _ = oc.oc_update(x, g, P.T @ np.ones(n), P, 0.3, 0.2, 0.5)
    assert steps > 0 and np.ptp(xn) == 0.0
    assert math.isclose(xn.mean(), 0.3, rel_tol=1e-12)
    # closed form: 0.35 sqrt(2/lam) = 0.3 -> lam = 2 (0.35/0.3)^2
    assert math.isclose(lam, 2 * (0.35 / 0.3) ** 2, rel_tol=1e-12)


def test_oc_unreachable_and_zero_gradient():
    n = 4 * 3 * 2
    P = filt.filter_matrix(4, 3, 2, 1.0)
    x = np.full(n, 0.9)
    # g = 0 -> x_new = max(0, x - m) for any lambda; volume 0.7 n > 0.3 n target -> unreachable
    xn, lam, steps, _ = oc.oc_update(x, np.zeros(n), np.ones(n), P, 0.3, 0.2, 0.5)
    assert steps < 0 and np.allclose(xn, 0.7)


# ------------------------------------------------------------------ loop
def test_simp_loop_makes_progress():
    # the standard run decreases compliance from the uniform start
    p = inputs.Problem("loop", 12, 6, 6, rmin=1.5)
    op = OracleProblem(p)
    h = simp_loop(op, np.full(p.n_elem, p.volfrac), 8, direct=True)
    assert h["c"][-1] < h["c"][0]
    assert all(s > 0 for s in h["steps"][1:])
    xf = h["x_final"]
    assert abs(np.sum(op.P @ xf) - p.volfrac * p.n_elem) <= 1e-8 * p.n_elem


def test_filter_rows_match_the_full_matrix():
    """oracle.filt.filter_rows / hs_of (element-by-element P x, P^T v for grids too large for
    the full matrix) agree with filter_matrix on a small grid, forward and transpose."""
    nx, ny, nz, rmin = 9, 7, 6, 2.6
    P = filt.filter_matrix(nx, ny, nz, rmin)
    _, Hs = filt.filter_matrices(nx, ny, nz, rmin)
    x = np.random.default_rng(3).uniform(0, 1, nx * ny * nz)
    elems = np.arange(0, nx * ny * nz, 7)
    assert np.allclose(filt.hs_of(nx, ny, nz, rmin, elems), Hs[elems], rtol=1e-14, atol=0)
    assert np.allclose(filt.filter_rows(nx, ny, nz, rmin, elems, x), (P @ x)[elems], rtol=1e-13, atol=0)
    assert np.allclose(filt.filter_rows(nx, ny, nz, rmin, elems, x, transpose=True), (P.T @ x)[elems],
                       rtol=1e-13, atol=0)
