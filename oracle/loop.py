"""One exact-gradient evaluation and the SIMP loop (oracle; test infrastructure only).

Cites: Eq. (2) (NAND: u(z) solved at every iteration)
Alg. 1 lines 8-9 ("solve r(z,u) = 0", "get exact gradients") and line 13
("update z with g"); Eq. (4)-(5); SPEC:531-539 [OP run_standard];
SURVEY §8 a10 and readings A6 (loops solve with rho~ = P x; single evaluations take
rho directly), A12 (parity solves start from x0 = 0), A18 (c_k recorded at x_k).
"""
from __future__ import annotations

import numpy as np

from . import fem, filt, grid, oc, sens, solve


class OracleProblem:
    """Everything the oracle needs for one problem description (inputs.Problem-like)."""

    def __init__(self, p, assemble=True):
        self.p = p
        nx, ny, nz = p.nx, p.ny, p.nz
        self.n_e, self.n_n, self.n_dof = grid.counts(nx, ny, nz)
        self.edof = grid.element_dofs(nx, ny, nz)
        self.KE = fem.element_stiffness(p.nu, p.h)
        self.fixed, self.load_dofs, self.load_vals = grid.bc_for(p.bc, nx, ny, nz, p.load_total)
        self.f = grid.load_vector(self.n_dof, self.load_dofs, self.load_vals)
        self._assemble = assemble
        self._P = None

    # ---- operator -------------------------------------------------------
    def E(self, rho):
        return fem.simp(rho, self.p.E0, self.p.Emin, self.p.penal)

    def Khat(self, rho):
        K = fem.assemble(self.edof, self.E(rho), self.KE, self.n_dof)
        return fem.apply_bc(K, self.fixed)

    def apply(self, rho, u):
        return fem.apply_matfree(u, self.E(rho), self.KE, self.edof, self.fixed)

    def dinv(self, rho):
        return 1.0 / fem.jacobi_diag(self.E(rho), self.KE, self.edof, self.fixed)

    # ---- solves ---------------------------------------------------------
    def solve_direct(self, rho):
        return solve.direct_solve(self.Khat(rho), self.f)

    def solve_pcg(self, rho, tol=1e-10, max_iters=200000, x0=None, use_csr=None, callback=None,
                  callback_u=None):
        E = self.E(rho)
        if use_csr is None:
            use_csr = self._assemble and self.n_e <= 120_000
        if use_csr:
            A = fem.apply_bc(fem.assemble(self.edof, E, self.KE, self.n_dof), self.fixed)
            op = A.__matmul__
        else:
            def op(v):
                return fem.apply_matfree(v, E, self.KE, self.edof, self.fixed)
        dinv = 1.0 / fem.jacobi_diag(E, self.KE, self.edof, self.fixed)
        return solve.pcg(op, dinv, self.f, x0=x0, tol=tol, max_iters=max_iters, callback=callback,
                         callback_u=callback_u)

    # ---- gradient pieces ------------------------------------------------
    @property
    def P(self):
        if self._P is None:
            self._P = filt.filter_matrix(self.p.nx, self.p.ny, self.p.nz, self.p.rmin)
        return self._P

    def compliance(self, u):
        return sens.compliance(self.f, u)

    def sensitivity(self, rho, u):
        return sens.sensitivity(rho, u, self.KE, self.edof, self.p.E0, self.p.Emin,
                                self.p.penal, self.fixed)

    def evaluate(self, rho, u):
        """Given the state u: (c, dc, ce, P^T dc) -- Eq. (4), Eq. (5), density-filter chain rule."""
        c = self.compliance(u)
        dc, ce = self.sensitivity(rho, u)
        return c, dc, ce, filt.apply_transpose(self.P, dc)

    def oc(self, x, g):
        dv = filt.volume_gradient(self.P)
        return oc.oc_update(x, g, dv, self.P, self.p.volfrac, self.p.move, self.p.eta)


def simp_loop(op: OracleProblem, x0, iters, tol=1e-10, direct=False, record_x=False):
    """SIMP/OC loop: for k: rho~ = P x_k; solve (x0 = 0); c_k; dc~; g = P^T dc~;
    x_{k+1} = OC(x_k, g).  Returns dict of histories."""
    x = np.array(x0, dtype=np.float64)
    hist = {"c": [], "lam": [], "steps": [], "iters": [], "x": []}
    for _ in range(iters):
        rho = filt.apply(op.P, x)
        if direct:
            u = op.solve_direct(rho)
            its = 0
        else:
            u, its, conv, _ = op.solve_pcg(rho, tol=tol)
            assert conv
        c, dc, _, g = op.evaluate(rho, u)
        xn, lam, steps, _ = op.oc(x, g)
        hist["c"].append(c)
        hist["lam"].append(lam)
        hist["steps"].append(steps)
        hist["iters"].append(its)
        if record_x:
            hist["x"].append(x.copy())
        x = xn
    hist["x_final"] = x
    return hist
