"""GPU error paths and solver-control semantics against the oracle (SPEC.md l.169-177 [OP pcg]:
"p^T K p <= 0 -> breakdown error", l.172 max_iters is not an error; l.318-335 [OP oc_update]:
"NaN in gradients -> error"; l.118: densities outside [0,1] are a domain error), plus the
two PCG loop executions (CUDA graph / host-batched) agreeing bit for bit."""
import numpy as np
import pytest
import torch

from oracle import fem, filt, oc as ooc
from oracle.loop import OracleProblem
from paper_2104_12282_b200 import inputs, tomo

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def gpu(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def test_breakdown_on_singular_translation_load():
    """One element, nothing fixed (K_hat = K, singular: the 6 rigid modes) and the same x load
    on all 8 nodes. All 8 nodes carry the same diagonal, so z_0 = D^-1 f is an exact
    x-translation t and p_0^T K p_0 = 0: "p^T K p <= 0 -> breakdown error".
    The GPU core sees only differences of corner values, which are exactly 0 for t, so the
    breakdown is exact there; the oracle's assembled K annihilates t only to rounding
    (its row sums are ~1e-17), which the test pins instead."""
    KE = fem.element_stiffness(0.3)
    t_x = np.tile([1.0, 0.0, 0.0], 8)
    assert abs(t_x @ KE @ t_x) <= 1e-14 * (t_x @ np.diag(np.diag(KE)) @ t_x)
    dofs = tuple(3 * n for n in range(8))
    p = tomo.Params(1, 1, 1, bc=tomo.TOMO_BC_EXPLICIT, load_dofs=dofs, load_vals=(0.125,) * 8)
    t = tomo.Tomo(p, device=DEV)
    with pytest.raises(tomo.TomoError) as ei:
        t.solve(gpu(np.ones(1)))
    assert ei.value.code == -4  # TOMO_EBREAKDOWN


def test_nonfinite_initial_guess_is_enan():
    p, rho = inputs.random_problem(8, 5, 4, seed=3)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u0 = np.zeros(p.n_dof)
    u0[3 * 40 + 1] = np.inf  # a free DOF (node 40 is not on the clamped face)
    with pytest.raises(tomo.TomoError) as ei:
        t.solve(gpu(rho), u=gpu(u0))
    assert ei.value.code == -6  # TOMO_ENAN
    u0[3 * 40 + 1] = np.nan
    with pytest.raises(tomo.TomoError) as ei:
        t.solve(gpu(rho), u=gpu(u0))
    assert ei.value.code == -6
    # the context stays usable after the error
    u, info = t.solve(gpu(rho))
    assert info.converged >= 1


def test_nan_density_is_domain_error():
    p, rho = inputs.random_problem(5, 3, 2, seed=4)
    rho[7] = np.nan
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    with pytest.raises(tomo.TomoError) as ei:
        t.solve(gpu(rho))
    assert ei.value.code == -2  # TOMO_EDOMAIN
    with pytest.raises(ValueError):
        OracleProblem(p).E(rho)


@pytest.mark.parametrize("which", ["g", "x", "dv"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_oc_nonfinite_inputs_are_enan(which, bad):
    nx, ny, nz = 6, 5, 4
    p = inputs.Problem("o", nx, ny, nz)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    P = filt.filter_matrix(nx, ny, nz, 1.5)
    dv = filt.volume_gradient(P)
    rng = np.random.default_rng(1)
    x = rng.uniform(0.1, 0.9, p.n_elem)
    g = -rng.uniform(0, 1, p.n_elem)
    arrs = {"x": x.copy(), "g": g.copy(), "dv": dv.copy()}
    arrs[which][17] = bad
    with pytest.raises(ValueError):
        ooc.oc_update(arrs["x"], arrs["g"], arrs["dv"], P, 0.3)
    with pytest.raises(tomo.TomoError) as ei:
        t.oc_update(gpu(arrs["x"]), gpu(arrs["g"]), gpu(arrs["dv"]), 0.3)
    assert ei.value.code == -6  # TOMO_ENAN
    xn, lam, steps = t.oc_update(gpu(x), gpu(g), gpu(dv), 0.3)  # usable afterwards
    assert np.isfinite(lam)


@pytest.mark.parametrize("cfg", ["cfg0", "cfg2"])
def test_converged_flag_matches_true_residual(cfg):
    """converged = 1 iff the recursive AND the true residual met tol, 2 if only the recursive
    one did (include/tomo.h)."""
    p = inputs.CONFIGS[cfg]
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    for tol in (1e-6, 1e-10):
        _, info = t.solve(gpu(inputs.density_for(cfg)), tol=tol)
        assert info.rel_res_recursive <= tol
        assert info.converged == (1 if info.rel_res_true <= tol else 2), info.as_dict()


def test_graph_and_host_batched_loops_bit_identical():
    p = inputs.CFG0
    rho = gpu(inputs.density_for("cfg0"))
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u1, c1, dcf1, i1 = t.evaluate(rho)
    t.set_graph(False)
    l0 = t.launches
    u2, c2, dcf2, i2 = t.evaluate(rho)
    assert t.launches - l0 >= i2.iterations + 1
    t.set_graph(True)
    u3, c3, dcf3, i3 = t.evaluate(rho)
    assert i1.iterations == i2.iterations == i3.iterations and c1 == c2 == c3
    assert torch.equal(u1, u2) and torch.equal(u1, u3) and torch.equal(dcf1, dcf2)


@pytest.mark.parametrize("graph", [True, False])
def test_programmatic_launch_bit_identical(graph, monkeypatch):
    """Programmatic dependent launch (griddepcontrol.wait / launch_dependents,
    16 PDL-chained launches per WHILE body) only changes when blocks are scheduled: the
    iterates, count and residual history equal those of launch-to-launch order (TOMO_NO_PDL,
    read at bind), in the graph and in host batches; max_iters not a multiple of the body."""
    p = inputs.CFG2
    rho = gpu(inputs.density_for("cfg2"))
    out = []
    for pdl in (True, False):
        if pdl:
            monkeypatch.delenv("TOMO_NO_PDL", raising=False)
        else:
            monkeypatch.setenv("TOMO_NO_PDL", "1")
        t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
        t.set_graph(graph)
        h = t.set_history(600)
        u, info = t.solve(rho, tol=1e-10, max_iters=200000)
        u7, info7 = t.solve(rho, tol=1e-10, max_iters=37)
        out.append((u.clone(), info, h.clone(), u7.clone(), info7))
        t.close()
    (u1, i1, h1, v1, j1), (u2, i2, h2, v2, j2) = out
    assert i1.iterations == i2.iterations and i1.converged == i2.converged >= 1
    assert torch.equal(u1, u2) and torch.equal(h1, h2)
    assert j1.iterations == j2.iterations == 37 and j1.converged == 0 and torch.equal(v1, v2)


@pytest.mark.parametrize("cfg", ["cfg0", "cfg2"])
def test_exact_beta_variant_matches_textbook_count(cfg):
    """tomo_set_pcg_exact_beta(1): beta from the explicit r_{k+1} - the textbook recurrence of
    oracle.solve.pcg. Its iteration count matches the oracle's textbook count
    (recorded in the golden) to 2%, and its solution the single-pass one to the tolerance."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", f"{cfg}_solve.json")) as f:
        meta = json.load(f)
    p = inputs.CONFIGS[cfg]
    rho = gpu(inputs.density_for(cfg))
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    u1, i1 = t.solve(rho, tol=1e-10)
    t.set_pcg_exact_beta(True)
    u2, i2 = t.solve(rho, tol=1e-10)
    t.set_graph(False)
    u3, i3 = t.solve(rho, tol=1e-10)
    assert i2.converged >= 1 and i2.iterations == i3.iterations and torch.equal(u2, u3)
    k_ref = meta["pcg_iters_1e-10"]
    assert abs(i2.iterations - k_ref) <= max(3, 0.02 * k_ref), (i2.iterations, k_ref)
    d = float(torch.linalg.norm(u1 - u2) / torch.linalg.norm(u1))
    assert d <= 1e-8, d


def test_residual_history_trace():
    """tomo_set_history: launch k records r_k^T r_k; its last entry is the reported recursive
    residual, its first ||f||^2 (x0 = 0), and the trace is the same in graph and host-batched
    execution."""
    p, rho = inputs.random_problem(10, 6, 5, seed=8)
    t = tomo.Tomo(tomo.params_from_problem(p), device=DEV)
    h = t.set_history(2000)
    u, info = t.solve(gpu(rho), tol=1e-10)
    hh = h.cpu().numpy()[: info.iterations + 1]
    fn = float(np.sqrt((p.ny + 1) * (1.0 / (p.ny + 1)) ** 2))  # cantilever: -1 in ny+1 parts
    assert abs(np.sqrt(hh[0]) - fn) <= 1e-14 * fn
    assert abs(np.sqrt(hh[-1]) / fn - info.rel_res_recursive) <= 1e-14
    assert np.sqrt(hh[-1]) / fn <= 1e-10 and np.all(np.sqrt(hh[:-1]) / fn > 1e-10)
    t.set_graph(False)
    h2 = t.set_history(2000)
    t.solve(gpu(rho), tol=1e-10)
    assert np.array_equal(h2.cpu().numpy()[: info.iterations + 1], hh)
    t.set_history(0)
