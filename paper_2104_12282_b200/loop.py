"""SIMP/OC loop over the C ABI (Alg. 1
lines 8-9 and 13 with exact gradients at every iteration).

Orchestration only: every arithmetic step runs in libtomo's kernels.
    rho~ = P x_k                      tomo_filter(transpose=0)      (reading A6)
    u, c_k, dc~, g = P^T dc~          tomo_evaluate (x0 = 0, A12)
    x_{k+1} = OC(x_k, g, dv)          tomo_oc_update (A17), dv = P^T 1
"""
from __future__ import annotations

import torch

from .tomo import Tomo


class SimpLoop:
    def __init__(self, t: Tomo, volfrac: float, move: float = 0.2, eta: float = 0.5,
                 tol: float = 1e-10, max_iters: int = 50000, warm_start: bool = False):
        # warm_start: each solve starts from the previous iteration's u instead of x0 = 0
        # (reading A12 fixes x0 = 0 for parity runs, so the default is a cold start)
        self.warm_start = warm_start
        self.t = t
        self.volfrac, self.move, self.eta = volfrac, move, eta
        self.tol, self.max_iters = tol, max_iters
        self.dv = t.volume_grad()
        self.rho = t.zeros_elem()
        self.u = t.zeros_dof()
        self.dc = t.zeros_elem()
        self.g = t.zeros_elem()
        self.xn = t.zeros_elem()

    def step(self, x: torch.Tensor):
        """One iteration from x_k: returns (x_{k+1}, c_k, lambda_k, oc_steps, pcg_info)."""
        self.t.filter(x, out=self.rho)
        if not self.warm_start:
            with torch.cuda.stream(self.t.stream):  # the stream the library reads u on
                self.u.zero_()
        _, c, _, info = self.t.evaluate(self.rho, self.u, self.dc, self.g, tol=self.tol,
                                         max_iters=self.max_iters)
        xn, lam, steps = self.t.oc_update(x, self.g, self.dv, self.volfrac, self.move, self.eta,
                                          out=self.xn)
        return xn.clone(), c, lam, steps, info

    def run(self, x0: torch.Tensor, iters: int):
        x = x0.clone()
        hist = {"c": [], "lam": [], "steps": [], "iters": []}
        for _ in range(iters):
            x, c, lam, steps, info = self.step(x)
            hist["c"].append(c)
            hist["lam"].append(lam)
            hist["steps"].append(steps)
            hist["iters"].append(info.iterations)
        hist["x_final"] = x
        return hist
