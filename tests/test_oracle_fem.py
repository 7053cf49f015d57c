"""Pins of the oracle's grid / KE / operator / solve against closed forms, exact
arithmetic and textbook results (not against itself).  CPU only."""
import math
import os
import json

import numpy as np
import pytest
import sympy as sy

from oracle import fem, grid, solve
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ grid
def test_counts_spec_examples():
    # SPEC:41-43 [OP build_grid] examples
    assert grid.counts(1, 1, 1) == (1, 8, 24)
    assert grid.counts(2, 1, 1) == (2, 12, 36)
    n_e, _, n_dof = grid.counts(40, 20, 20)
    assert n_e == 16000 and n_dof == 54243
    # SURVEY §8 size table (App. B-1: the dimensions govern)
    assert grid.counts(24, 12, 12)[2] == 12675
    assert grid.counts(224, 112, 56)[2] == 4347675
    assert grid.counts(256, 128, 128)[2] == 12830211


def test_element_dofs_spec_examples():
    ed = grid.element_dofs(1, 1, 1)
    assert sorted(ed[0].tolist()) == list(range(24))
    ed = grid.element_dofs(2, 1, 1)
    assert len(set(ed[0]) & set(ed[1])) == 12  # SPEC:50 shared face
    for dims in [(3, 3, 3), (5, 3, 7), (1, 4, 1)]:  # SPEC:51 full cover + 24 distinct per element
        ed = grid.element_dofs(*dims)
        assert all(len(set(r)) == 24 for r in ed)
        assert set(ed.ravel()) == set(range(grid.counts(*dims)[2]))


def test_element_dofs_bruteforce_geometry():
    # corner a of element (i,j,k) sits at node (i+ax, j+ay, k+az), x fastest
    nx, ny, nz = 3, 2, 2
    ed = grid.element_dofs(nx, ny, nz)
    e = 0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                for a, (ax, ay, az) in enumerate(grid.CORNERS):
                    n = (i + ax) + (nx + 1) * ((j + ay) + (ny + 1) * (k + az))
                    assert ed[e, 3 * a:3 * a + 3].tolist() == [3 * n, 3 * n + 1, 3 * n + 2]
                e += 1


def test_cantilever_preset():
    fixed, dofs, vals = grid.cantilever_bc(4, 2, 2, -1.0)
    assert fixed.sum() == 27
    assert math.isclose(vals.sum(), -1.0, rel_tol=1e-15)  # BASELINE configs[0]: total load -1
    assert not fixed[dofs].any()
    assert (dofs % 3 == 2).all()
    # SURVEY size table: fixed DOFs / loaded nodes
    f3, d3, _ = grid.cantilever_bc(224, 112, 56)
    assert f3.sum() == 19323 and d3.size == 113


def test_mbb_half_preset():
    fixed, dofs, vals = grid.mbb_half_bc(96, 32, 32)
    assert fixed.sum() == 1123  # 1089 u_x + 33 u_z + 1 u_y (SURVEY size-table note)
    assert dofs.size == 33 and math.isclose(vals.sum(), -1.0)
    assert not fixed[dofs].any()


def _decode(dofs, nx, ny):
    """DOF -> (i, j, k, c) by the numbering of SPEC:26/30 (x fastest)."""
    out = []
    for d in np.asarray(dofs).tolist():
        n, c = divmod(d, 3)
        i = n % (nx + 1)
        j = (n // (nx + 1)) % (ny + 1)
        k = n // ((nx + 1) * (ny + 1))
        out.append((i, j, k, c))
    return out


@pytest.mark.parametrize("dims", [(5, 3, 4), (2, 1, 1), (7, 4, 2)])
def test_cantilever_preset_locations(dims):
    """Exact DOF sets of the cantilever preset, written from the text of BASELINE.json
    configs[0] ("x=0 face fully clamped; total load -1 in z spread evenly over the nodes of
    the bottom edge of the x=max face"; reading A8): fixed = every DOF of every node with
    i = 0; loaded = the z DOF of the nodes (nx, j, 0), j = 0..ny, each -1/(ny+1)."""
    nx, ny, nz = dims
    fixed, dofs, vals = grid.cantilever_bc(nx, ny, nz, -1.0)
    want_fixed = {(0, j, k, c) for j in range(ny + 1) for k in range(nz + 1) for c in range(3)}
    assert set(_decode(np.flatnonzero(fixed), nx, ny)) == want_fixed
    assert sorted(_decode(dofs, nx, ny)) == [(nx, j, 0, 2) for j in range(ny + 1)]
    assert np.all(vals == -1.0 / (ny + 1))


@pytest.mark.parametrize("dims", [(5, 3, 4), (4, 2, 2), (3, 1, 5)])
def test_mbb_half_preset_locations(dims):
    """Exact DOF sets of the MBB half-beam preset from BASELINE.json configs[2] ("symmetry
    (u_x=0) on the x=0 face, roller (u_z=0) on the bottom edge line at x=max, unit -z line
    load on the top edge at x=0") plus reading A9's u_y pin at node (nx, 0, 0) and A10's
    equal weights: fixed = {(0,j,k,x)} U {(nx,j,0,z)} U {(nx,0,0,y)}; loaded = {(0,j,nz,z)}."""
    nx, ny, nz = dims
    fixed, dofs, vals = grid.mbb_half_bc(nx, ny, nz, -1.0)
    want = {(0, j, k, 0) for j in range(ny + 1) for k in range(nz + 1)}
    want |= {(nx, j, 0, 2) for j in range(ny + 1)}
    want |= {(nx, 0, 0, 1)}
    assert set(_decode(np.flatnonzero(fixed), nx, ny)) == want
    assert sorted(_decode(dofs, nx, ny)) == [(0, j, nz, 2) for j in range(ny + 1)]
    assert np.all(vals == -1.0 / (ny + 1))


def test_mbb_half_equals_mirrored_full_beam():
    """Physics pin of the MBB half-beam preset, independent of grid.mbb_half_bc: the full
    simply supported beam of PAPER:207 ("MBB beam", load at the top centre), 2nx long,
    rollers u_z = 0 on the bottom edge lines x' = 0 and x' = 2nx, line load -2 on the top
    centre line x' = nx, rigid motions removed symmetrically (u_x at (nx,0,0), u_y at
    (0,0,0) and (2nx,0,0)). By mirror symmetry its right half x' = nx + x is the half-beam
    with u_x = 0 on the symmetry plane, the roller at x = nx, load -1 at x = 0 and the u_y
    pin at (nx,0,0) - so u agrees node by node and c_full = 2 c_half. A load on the wrong
    edge, a roller at x = 0 or the u_y pin at (0,0,0) all fail this."""
    nx, ny, nz = 4, 2, 3
    half = OracleProblem(inputs.Problem("half", nx, ny, nz, bc=inputs.BC_MBB_HALF))
    rng = np.random.default_rng(7)
    rho_half = rng.uniform(0.3, 1.0, half.n_e).reshape(nz, ny, nx)
    u_half = half.solve_direct(rho_half.ravel())
    # full beam: element (i', j, k) of the right half is the half's (i' - nx); left half mirrored
    NX = 2 * nx
    rho_full = np.concatenate([rho_half[:, :, ::-1], rho_half], axis=2).ravel()
    _, _, n_dof = grid.counts(NX, ny, nz)
    nid = lambda i, j, k: i + (NX + 1) * (j + (ny + 1) * k)  # noqa: E731
    fixed = np.zeros(n_dof, dtype=bool)
    for j in range(ny + 1):
        fixed[3 * nid(0, j, 0) + 2] = fixed[3 * nid(NX, j, 0) + 2] = True
    fixed[3 * nid(nx, 0, 0) + 0] = True
    fixed[3 * nid(0, 0, 0) + 1] = fixed[3 * nid(NX, 0, 0) + 1] = True
    f = np.zeros(n_dof)
    for j in range(ny + 1):
        f[3 * nid(nx, j, nz) + 2] = -2.0 / (ny + 1)
    KE = fem.element_stiffness(0.3)
    E = fem.simp(rho_full, 1.0, 1e-9, 3.0)
    K = fem.apply_bc(fem.assemble(grid.element_dofs(NX, ny, nz), E, KE, n_dof), fixed)
    u_full = solve.direct_solve(K, f)
    assert math.isclose(f @ u_full, 2.0 * (half.f @ u_half), rel_tol=1e-10)
    uf = u_full.reshape(nz + 1, ny + 1, NX + 1, 3)[:, :, nx:, :]
    uh = u_half.reshape(nz + 1, ny + 1, nx + 1, 3)
    assert np.max(np.abs(uf - uh)) <= 1e-9 * np.max(np.abs(uh))


# ------------------------------------------------------------------ KE
@pytest.mark.parametrize("nu", [0.3, 0.25, 0.45])
def test_ke_closed_form(nu):
    KE = fem.element_stiffness(nu)
    lam, mu = fem.lame(1.0, nu)
    # SURVEY App. A-2 row 0 (independently derived closed forms)
    assert np.allclose(np.diag(KE), (lam + 4 * mu) / 9, rtol=1e-14, atol=0)
    assert math.isclose(KE[0, 1], (lam + mu) / 12, rel_tol=1e-13)
    assert math.isclose(KE[0, 3], -(lam + mu) / 9, rel_tol=1e-13)
    assert math.isclose(KE[0, 4], (lam - mu) / 12, rel_tol=1e-12, abs_tol=1e-16)
    assert math.isclose(KE[0, 18], -(lam / 36 + mu / 9), rel_tol=1e-13)
    assert np.abs(KE - KE.T).max() <= 1e-15
    # spectrum (SURVEY A-2 lists mu x8 at nu = 0.3, where lam/3 + mu/2 = mu coincides):
    # 0 x6, mu/6 x2, lam/18+2mu/9 x3, mu/2 x3, 2mu/3 x1, mu x5, lam/3+mu/2 x3, (3lam+2mu)/2 x1
    ev = np.sort(np.linalg.eigvalsh(KE))
    expect = np.sort([0.0] * 6 + [mu / 6] * 2 + [lam / 18 + 2 * mu / 9] * 3 + [mu / 2] * 3
                     + [2 * mu / 3] + [mu] * 5 + [lam / 3 + mu / 2] * 3 + [(3 * lam + 2 * mu) / 2])
    assert np.allclose(ev, expect, atol=1e-13)


def test_ke_rigid_body_null_space():
    KE = fem.element_stiffness(0.3)
    X = np.array(grid.CORNERS, dtype=float)
    modes = []
    for c in range(3):  # translations
        t = np.zeros((8, 3)); t[:, c] = 1.0; modes.append(t.ravel())
    for a, b in [(0, 1), (1, 2), (2, 0)]:  # infinitesimal rotations
        r = np.zeros((8, 3)); r[:, a] = -X[:, b]; r[:, b] = X[:, a]; modes.append(r.ravel())
    for m in modes:
        assert np.abs(KE @ m).max() <= 1e-15
    assert np.linalg.matrix_rank(KE, tol=1e-9 * np.abs(KE).max()) == 18  # nullity 6


def test_ke_scales_with_h():
    assert np.allclose(fem.element_stiffness(0.3, h=2.5), 2.5 * fem.element_stiffness(0.3), rtol=1e-14)


def _ke_exact_sympy(nu):
    """KE by exact symbolic integration over the unit cube (independent of the Gauss path)."""
    x, y, z = sy.symbols("x y z")
    nu = sy.Rational(nu)
    lam = nu / ((1 + nu) * (1 - 2 * nu))
    mu = 1 / (2 * (1 + nu))
    N = []
    for ax, ay, az in grid.CORNERS:
        N.append((x if ax else 1 - x) * (y if ay else 1 - y) * (z if az else 1 - z))
    grads = [[sy.diff(n, v) for v in (x, y, z)] for n in N]
    K = sy.zeros(24, 24)
    for a in range(8):
        for b in range(8):
            for c in range(3):
                for d in range(3):
                    # KE[(a,c),(b,d)] = int lam dcNa ddNb + mu ddNa dcNb + mu delta_cd gradNa.gradNb
                    expr = lam * grads[a][c] * grads[b][d] + mu * grads[a][d] * grads[b][c]
                    if c == d:
                        expr += mu * sum(grads[a][q] * grads[b][q] for q in range(3))
                    K[3 * a + c, 3 * b + d] = sy.integrate(sy.expand(expr), (x, 0, 1), (y, 0, 1), (z, 0, 1))
    return K


def _exact_cantilever_compliance(nx, KE):
    p = inputs.Problem("g", nx, 1, 1)
    op = OracleProblem(p)
    n = op.n_dof
    K = sy.zeros(n, n)
    for e in range(op.n_e):
        d = op.edof[e]
        for r in range(24):
            for s in range(24):
                K[d[r], d[s]] += KE[r, s]
    free = [i for i in range(n) if not op.fixed[i]]
    f = sy.zeros(n, 1)
    for dof, _ in zip(op.load_dofs, op.load_vals):
        f[int(dof)] += sy.Rational(-1, 2)
    Kf = K.extract(free, free)
    ff = f.extract(free, [0])
    u = Kf.LUsolve(ff)
    return sy.nsimplify((ff.T * u)[0])


@pytest.mark.slow
def test_golden_tiny_cantilever_exact():
    """Exact-rational compliance of 1x1x1 and 2x1x1 clamped cantilevers,
    re-derived here in exact arithmetic, against the oracle's float pipeline."""
    with open(os.path.join(GOLDEN, "tiny_cantilever.json")) as fh:
        gold = json.load(fh)
    KE = _ke_exact_sympy("3/10")
    for case in gold["cases"]:
        nx = case["nx"]
        exact = _exact_cantilever_compliance(nx, KE)
        assert exact == sy.Rational(case["num"], case["den"])
        p = inputs.Problem("g", nx, 1, 1)
        op = OracleProblem(p)
        u = op.solve_direct(np.ones(p.n_elem))
        assert math.isclose(op.compliance(u), float(exact), rel_tol=1e-13)
    # the exact KE also equals the quadrature KE
    assert np.allclose(np.array(KE, dtype=float), fem.element_stiffness(0.3), rtol=1e-14, atol=1e-16)


def test_uniform_density_scaling():
    # c(rho) = c(1) E0 / E(rho) at uniform rho (SURVEY A-4)
    p = inputs.Problem("g", 3, 2, 2)
    op = OracleProblem(p)
    c1 = op.compliance(op.solve_direct(np.ones(p.n_elem)))
    rho = 0.4
    Er = p.Emin + rho ** 3 * (p.E0 - p.Emin)
    c = op.compliance(op.solve_direct(np.full(p.n_elem, rho)))
    assert math.isclose(c, c1 / Er, rel_tol=1e-11)


# ------------------------------------------------------------------ operator
def _dense_bruteforce(nx, ny, nz, E, KE, fixed):
    n = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    K = np.zeros((n, n))
    e = 0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                d = []
                for ax, ay, az in grid.CORNERS:
                    nd = (i + ax) + (nx + 1) * ((j + ay) + (ny + 1) * (k + az))
                    d += [3 * nd, 3 * nd + 1, 3 * nd + 2]
                for r in range(24):
                    for s in range(24):
                        K[d[r], d[s]] += E[e] * KE[r, s]
                e += 1
    for q in range(n):
        if fixed[q]:
            K[q, :] = 0.0
            K[:, q] = 0.0
            K[q, q] = 1.0
    return K


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (2, 2, 3), (3, 3, 3)])
def test_apply_matches_bruteforce_dense(dims):
    # apply agrees with dense assembly up to 3x3x3 at 1e-10
    p, rho = inputs.random_problem(*dims, seed=7)
    op = OracleProblem(p)
    E = op.E(rho)
    Kd = _dense_bruteforce(*dims, E, op.KE, op.fixed)
    u = inputs.random_vector(op.n_dof, 3)
    y = op.apply(rho, u)
    assert np.abs(y - Kd @ u).max() <= 1e-12 * np.abs(Kd @ u).max()
    assert np.abs(op.Khat(rho).toarray() - Kd).max() <= 1e-15
    assert np.allclose(1.0 / op.dinv(rho), np.diag(Kd), rtol=1e-15)


def test_apply_identities():
    p, rho = inputs.random_problem(4, 3, 2, seed=1)
    op = OracleProblem(p)
    u = inputs.random_vector(op.n_dof, 1)
    v = inputs.random_vector(op.n_dof, 2)
    assert np.abs(op.apply(rho, np.zeros(op.n_dof))).max() == 0.0
    assert np.allclose(op.apply(rho, 2.5 * u), 2.5 * op.apply(rho, u), rtol=1e-13)
    assert math.isclose(v @ op.apply(rho, u), u @ op.apply(rho, v), rel_tol=1e-12)  # symmetry
    uf = np.where(op.fixed, 0.0, u)
    assert uf @ op.apply(rho, uf) > 0.0  # SPEC:144 energy positivity


def test_linear_field_interior_zero_and_patch():
    """SURVEY A-3: uniform E, no BCs: K u_lin = 0 at interior nodes; u_x = eps x gives
    ce = (lam + 2 mu) eps^2 h^3 per element (uniaxial strain)."""
    nx, ny, nz = 4, 3, 3
    op = OracleProblem(inputs.Problem("g", nx, ny, nz))
    fixed = np.zeros(op.n_dof, dtype=bool)
    E = np.ones(op.n_e)
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    X = np.stack([i.ravel(), j.ravel(), k.ravel()], 1).astype(float)
    A = np.array([[0.3, -0.2, 0.1], [0.05, 0.4, -0.3], [0.2, 0.1, -0.1]])
    u = (X @ A.T).ravel()
    y = fem.apply_matfree(u, E, op.KE, op.edof, fixed)
    interior = ((X[:, 0] > 0) & (X[:, 0] < nx) & (X[:, 1] > 0) & (X[:, 1] < ny)
                & (X[:, 2] > 0) & (X[:, 2] < nz))
    assert np.abs(y.reshape(-1, 3)[interior]).max() <= 1e-14
    lam, mu = fem.lame(1.0, 0.3)
    ux = np.zeros((op.n_n, 3)); ux[:, 0] = X[:, 0]
    from oracle import sens
    ce = sens.element_energy(ux.ravel(), op.KE, op.edof)
    assert np.allclose(ce, lam + 2 * mu, rtol=1e-14)
    assert math.isclose(lam + 2 * mu, 1.3461538461538463, rel_tol=1e-15)


def test_dirichlet_patch_test():
    """Linear u prescribed on all boundary nodes reproduces the linear field inside (~1e-13)."""
    nx, ny, nz = 4, 4, 3
    op = OracleProblem(inputs.Problem("g", nx, ny, nz))
    k, j, i = np.meshgrid(np.arange(nz + 1), np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    X = np.stack([i.ravel(), j.ravel(), k.ravel()], 1).astype(float)
    A = np.array([[0.3, -0.2, 0.1], [0.05, 0.4, -0.3], [0.2, 0.1, -0.1]])
    ulin = (X @ A.T + np.array([0.1, -0.2, 0.3])).ravel()
    bnd = ((X[:, 0] == 0) | (X[:, 0] == nx) | (X[:, 1] == 0) | (X[:, 1] == ny)
           | (X[:, 2] == 0) | (X[:, 2] == nz))
    fixed = np.repeat(bnd, 3)
    K = fem.assemble(op.edof, np.ones(op.n_e), op.KE, op.n_dof).toarray()
    free = ~fixed
    rhs = -K[np.ix_(free, fixed)] @ ulin[fixed]
    uf = np.linalg.solve(K[np.ix_(free, free)], rhs)
    assert np.abs(uf - ulin[free]).max() <= 1e-13


# ------------------------------------------------------------------ solve
def test_pcg_toy_systems():
    # SPEC:175 identity -> 1 iteration; SPEC:176 [[4,1],[1,3]] f=(1,2) -> (1/11, 7/11)
    f = np.array([1.0, -2.0, 3.0])
    u, k, conv, _ = solve.pcg(lambda v: v, np.ones(3), f, tol=1e-12)
    assert k == 1 and conv and np.array_equal(u, f)
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    u, k, conv, _ = solve.pcg(lambda v: A @ v, 1.0 / np.diag(A), np.array([1.0, 2.0]), tol=1e-14)
    assert conv and np.allclose(u, [1 / 11, 7 / 11], rtol=1e-14)
    u, k, conv, _ = solve.pcg(lambda v: A @ v, np.ones(2), np.zeros(2))
    assert k == 0 and not u.any()
    with pytest.raises(solve.Breakdown):
        solve.pcg(lambda v: -v, np.ones(2), np.array([1.0, 1.0]))


def test_pcg_single_pass_toy_systems_and_finite_termination():
    """oracle.solve.pcg_single_pass (reading R1) against closed forms and CG theory: the
    identity needs 1 iteration; the 2x2 system of SPEC:176 gives (1/11, 7/11); on an SPD
    matrix with n distinct eigenvalues Krylov optimality terminates in n iterations, like
    textbook pcg; the breakdown rule holds."""
    f = np.array([1.0, -2.0, 3.0])
    u, k, conv, _ = solve.pcg_single_pass(lambda v: v, np.ones(3), f, tol=1e-12)
    assert k == 1 and conv and np.array_equal(u, f)
    A = np.array([[4.0, 1.0], [1.0, 3.0]])
    u, k, conv, _ = solve.pcg_single_pass(lambda v: A @ v, 1.0 / np.diag(A), np.array([1.0, 2.0]),
                                          tol=1e-14)
    assert conv and np.allclose(u, [1 / 11, 7 / 11], rtol=1e-14)
    rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    B = Q @ np.diag(np.linspace(1.0, 4.0, 8)) @ Q.T
    b = rng.standard_normal(8)
    x = np.linalg.solve(B, b)
    for fn in (solve.pcg, solve.pcg_single_pass):
        u, k, conv, _ = fn(lambda v: B @ v, np.ones(8), b, tol=1e-10)
        assert conv and k <= 8 and np.allclose(u, x, rtol=1e-9)
    with pytest.raises(solve.Breakdown):
        solve.pcg_single_pass(lambda v: -v, np.ones(2), np.array([1.0, 1.0]))


def test_pcg_single_pass_matches_textbook_fem():
    """On a moderately conditioned FE system the single-pass recurrence reproduces textbook
    Jacobi-PCG: the same iteration count (+-1) and the same solution to the tolerance."""
    p, rho = inputs.random_problem(8, 4, 4, seed=12, lo=0.2)
    op = OracleProblem(p)
    E = op.E(rho)
    K = op.Khat(rho)
    dinv = op.dinv(rho)
    u1, k1, c1, _ = solve.pcg(K.__matmul__, dinv, op.f, tol=1e-10)
    u2, k2, c2, _ = solve.pcg_single_pass(K.__matmul__, dinv, op.f, tol=1e-10)
    assert c1 and c2 and abs(k1 - k2) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-8 * np.linalg.norm(u1)
    assert E.size == p.n_elem


def test_pcg_matches_direct_fem():
    p, rho = inputs.random_problem(6, 3, 3, seed=11, lo=0.2)
    op = OracleProblem(p)
    ud = op.solve_direct(rho)
    u, k, conv, rr = op.solve_pcg(rho, tol=1e-12)
    assert conv and rr <= 1e-12
    assert np.linalg.norm(u - ud) <= 1e-10 * np.linalg.norm(ud)
    assert np.abs(op.apply(rho, ud) - op.f).max() <= 1e-10 * np.abs(op.f).max()


def _cantilever_end_face(n, nu=0.0):
    """Beam 16n x n x n, clamped x=0, end load total -1 on the x=L face with bilinear lumping;
    mean u_z on the end face."""
    nx, ny, nz = 16 * n, n, n
    p = inputs.Problem("eb", nx, ny, nz, nu=nu, Emin=0.0, E0=1.0)
    op = OracleProblem(p)
    w1 = np.array([0.5] + [1.0] * (n - 1) + [0.5]) / n  # trapezoid weights on [0, 1] edge of n cells
    W = np.outer(w1, w1)  # (k, j) weights summing to 1
    f = np.zeros(op.n_dof)
    face = []
    for k in range(nz + 1):
        for j in range(ny + 1):
            nd = nx + (nx + 1) * (j + (ny + 1) * k)
            f[3 * nd + 2] = -W[k, j]
            face.append(nd)
    u = __import__("scipy.sparse.linalg", fromlist=["spsolve"]).spsolve(op.Khat(np.ones(op.n_e)).tocsc(), f)
    return -np.mean(u[3 * np.array(face) + 2])


@pytest.mark.slow
def test_euler_bernoulli_refinement():
    """SURVEY A-7: delta_EB = F L^3/(3 E I) = 16384/n, Timoshenko + F L/(kappa G A) = 38.4/n.
    Fully integrated hex8 locks: delta_h < delta_T, increasing with n; Richardson from n=4,8
    within 2% of Timoshenko."""
    d = {n: _cantilever_end_face(n) for n in (2, 4, 8)}
    dT = {n: 16384.0 / n + 38.4 / n for n in d}
    scaled = {n: d[n] * n for n in d}  # n * delta is mesh-size independent for the exact beam
    assert scaled[2] < scaled[4] < scaled[8] < dT[8] * 8
    rich = scaled[8] + (scaled[8] - scaled[4]) / 3.0
    assert abs(rich - dT[8] * 8) / (dT[8] * 8) < 0.02
