"""Optimality-criteria design update (oracle; test infrastructure only).

Cites: PAPER:184 ("we use the optimality criteria (OC) method, which the
standard optimizer for (4), to update design variables z")
Eq. (4) (volume constraint v^T P z <= V_max, box 0 <= z_i <= 1)
[OP oc_update] z_new = clamp(z (-g/(lambda dV))^eta, max(0, z - m), min(1, z + m));
SURVEY reading A17 (canonical deterministic bisection):

    l1 = 1e-30, l2 = 1e30; while l2 > l1 (1 + 1e-15) and steps < 200:
        lm = sqrt(l1 l2); if V(x_new(lm)) > V*: l1 = lm else l2 = lm
    lambda = l2 (feasible side), output x_new(l2)

with V(x) = 1^T (P x) measured literally and V* = volfrac * N_e.  Positive g is
clamped to 0.  If the target is unreachable within the move limits the step
count is returned negated (not an error).
"""
from __future__ import annotations

import numpy as np


def x_new(x, g, dv, lam, move, eta):
    B = np.maximum(0.0, -g) / (dv * lam)
    scale = np.sqrt(B) if eta == 0.5 else B ** eta
    return np.clip(x * scale, np.maximum(0.0, x - move), np.minimum(1.0, x + move))


def oc_update(x, g, dv, P, volfrac, move=0.2, eta=0.5, l1=1e-30, l2=1e30, rel=1e-15,
              max_steps=200):
    """Returns (x_new, lambda, steps, flips_trace) -- steps < 0 if the target was unreachable.
    Non-finite x, g or dv raise ValueError ("NaN in gradients -> error")."""
    if not (np.all(np.isfinite(x)) and np.all(np.isfinite(g)) and np.all(np.isfinite(dv))):
        raise ValueError("NaN/Inf in x, g or dv (SPEC:322)")
    target = volfrac * x.size

    def vol(xx):
        return float(np.sum(P @ xx))

    lo0, hi0 = l1, l2
    steps = 0
    trace = []
    while l2 > l1 * (1.0 + rel) and steps < max_steps:
        lm = np.sqrt(l1 * l2)
        v = vol(x_new(x, g, dv, lm, move, eta))
        if v > target:
            l1 = lm
        else:
            l2 = lm
        trace.append((lm, v > target))
        steps += 1
    unreachable = (l2 == hi0) or (l1 == lo0)
    return x_new(x, g, dv, l2, move, eta), l2, (-steps if unreachable else steps), trace
