"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle (``oracle/``), the tests and ``bench.py``.
It holds NONE of the method's arithmetic (no stiffness, no filter, no solver,
no OC): only problem descriptions and seeded density fields, so that both the
CUDA path and the oracle consume bit-identical arrays.

Recipes follow SURVEY.md §8(d1) (the readings are listed in DESIGN.md §3):

* cfg0  24x12x12 cantilever, rho = 0.3 + U(-0.1, 0.1), seed 0      (BASELINE.json configs[0])
* cfg1  48x24x24 cantilever, x0 = 0.3 uniform, 50 SIMP/OC steps      (configs[1])
* cfg2  96x32x32 MBB half-beam, smooth seeded sine field, seed 2     (configs[2])
* cfg3  224x112x56 cantilever, blob / Beta(0.5,0.5) field, seed 3    (configs[3], the metric)
* cfg4  sweep grids, void-0.7 blobs (seed 4) or uniform 0.5          (configs[4])

Arrays are in element order e = i + nx*(j + ny*k) (x fastest), i.e. a
C-order array of shape (nz, ny, nx) raveled.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# BC kinds (mirrors tomo_bc_kind in include/tomo.h; plain integers, no arithmetic)
BC_CANTILEVER = 1
BC_MBB_HALF = 2
BC_EXPLICIT = 3


@dataclasses.dataclass(frozen=True)
class Problem:
    name: str
    nx: int
    ny: int
    nz: int
    bc: int = BC_CANTILEVER
    E0: float = 1.0
    Emin: float = 1e-9
    nu: float = 0.3
    penal: float = 3.0
    rmin: float = 1.5
    h: float = 1.0
    load_total: float = -1.0
    tol: float = 1e-10
    volfrac: float = 0.3
    move: float = 0.2
    eta: float = 0.5
    loop_iters: int = 0

    @property
    def n_elem(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_node(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_dof(self) -> int:
        return 3 * self.n_node


CFG0 = Problem("cfg0_cantilever_24x12x12", 24, 12, 12, rmin=1.5)
CFG1 = Problem("cfg1_cantilever_48x24x24_loop50", 48, 24, 24, rmin=1.5, loop_iters=50)
CFG2 = Problem("cfg2_mbb_half_96x32x32", 96, 32, 32, bc=BC_MBB_HALF, rmin=2.0)
CFG3 = Problem("cfg3_cantilever_224x112x56", 224, 112, 56, rmin=3.0, loop_iters=20)
CFG4_GRIDS = ((32, 32, 32), (64, 64, 64), (128, 64, 64), (192, 96, 96), (256, 128, 128))


def cfg4(idx: int) -> Problem:
    nx, ny, nz = CFG4_GRIDS[idx]
    return Problem(f"cfg4{'abcde'[idx]}_cantilever_{nx}x{ny}x{nz}", nx, ny, nz, rmin=1.5)


CONFIGS = {"cfg0": CFG0, "cfg1": CFG1, "cfg2": CFG2, "cfg3": CFG3}
for _i in range(5):
    CONFIGS[f"cfg4{'abcde'[_i]}"] = cfg4(_i)


# ---------------------------------------------------------------- densities
def _centroids(p: Problem):
    k, j, i = np.meshgrid(np.arange(p.nz), np.arange(p.ny), np.arange(p.nx), indexing="ij")
    return (i + 0.5).ravel(), (j + 0.5).ravel(), (k + 0.5).ravel()


def density_cfg0(p: Problem = CFG0, seed: int = 0) -> np.ndarray:
    """rho = 0.3 + U(-0.1, 0.1) per element (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    return 0.3 + rng.uniform(-0.1, 0.1, p.n_elem)


def density_uniform(p: Problem, value: float) -> np.ndarray:
    return np.full(p.n_elem, float(value))


def density_sines(p: Problem = CFG2, seed: int = 2, n_terms: int = 6) -> np.ndarray:
    """Smooth seeded field rho = clip(0.3 + 0.25*sum_k a_k sin(w_k.x + phi_k), 0.001, 1)
    (BASELINE.json configs[2]; draw order a, m, phi as in SURVEY §8 d1)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, n_terms)
    m = rng.integers(1, 5, size=(n_terms, 3))
    phi = rng.uniform(0.0, 2.0 * np.pi, n_terms)
    x, y, z = _centroids(p)
    s = np.zeros(p.n_elem)
    for t in range(n_terms):
        wx = 2.0 * np.pi * m[t, 0] / p.nx
        wy = 2.0 * np.pi * m[t, 1] / p.ny
        wz = 2.0 * np.pi * m[t, 2] / p.nz
        s += a[t] * np.sin(wx * x + wy * y + wz * z + phi[t])
    return np.clip(0.3 + 0.25 * s, 0.001, 1.0)


def _blur_axis(g: np.ndarray, sigma: float, axis: int) -> np.ndarray:
    """1-D Gaussian blur along one axis, truncated at 3 sigma, reflect boundary
    (input-recipe smoothing, not part of the method)."""
    r = int(math.ceil(3.0 * sigma))
    t = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (t / sigma) ** 2)
    w /= w.sum()
    n = g.shape[axis]
    pad = [(0, 0)] * g.ndim
    pad[axis] = (r, r)
    gp = np.pad(g, pad, mode="symmetric")
    out = np.zeros_like(g)
    for q, wq in enumerate(w):
        sl = [slice(None)] * g.ndim
        sl[axis] = slice(q, q + n)
        out += wq * gp[tuple(sl)]
    return out


def _blob_field(p: Problem, rng, sigma: float) -> np.ndarray:
    g = rng.standard_normal(p.n_elem).reshape(p.nz, p.ny, p.nx)
    for ax in range(3):
        g = _blur_axis(g, sigma, ax)
    return g.ravel()


def _forced_margin(p: Problem) -> np.ndarray:
    """Elements kept solid-ish: i < 2 (clamped face) and (i >= nx-2 and k < 2) (load edge)."""
    k, j, i = np.meshgrid(np.arange(p.nz), np.arange(p.ny), np.arange(p.nx), indexing="ij")
    m = (i < 2) | ((i >= p.nx - 2) & (k < 2))
    return m.ravel()


def density_blobs_beta(p: Problem = CFG3, seed: int = 3, void_frac: float = 0.3,
                       sigma: float = 6.0, void_value: float = 1e-3) -> np.ndarray:
    """Mid-optimisation-like field (BASELINE.json configs[3]): the lowest 30% of a
    blurred white-noise field are void (1e-3) in spatially correlated blobs, the
    rest Beta(0.5,0.5) = sin^2(pi U / 2)."""
    rng = np.random.default_rng(seed)
    g = _blob_field(p, rng, sigma)
    u = rng.uniform(0.0, 1.0, p.n_elem)
    rho = np.sin(0.5 * np.pi * u) ** 2
    order = np.argsort(g, kind="stable")
    void = np.zeros(p.n_elem, dtype=bool)
    void[order[: int(void_frac * p.n_elem)]] = True
    void &= ~_forced_margin(p)
    rho[void] = void_value
    return rho


def density_void07(p: Problem, seed: int = 4, sigma: float = 4.0) -> np.ndarray:
    """High-contrast sweep field (BASELINE.json configs[4]): lowest 70% of blurred
    noise -> rho = 0 (E = Emin), rest rho = 1, same forced margin."""
    rng = np.random.default_rng(seed)
    g = _blob_field(p, rng, sigma)
    order = np.argsort(g, kind="stable")
    rho = np.ones(p.n_elem)
    void = np.zeros(p.n_elem, dtype=bool)
    void[order[: int(0.7 * p.n_elem)]] = True
    void &= ~_forced_margin(p)
    rho[void] = 0.0
    return rho


def density_for(name: str, variant: Optional[str] = None) -> np.ndarray:
    p = CONFIGS[name]
    if name == "cfg0":
        return density_cfg0(p)
    if name == "cfg1":
        return density_uniform(p, p.volfrac)
    if name == "cfg2":
        return density_sines(p)
    if name == "cfg3":
        return density_blobs_beta(p)
    if name.startswith("cfg4"):
        if variant in (None, "void07"):
            return density_void07(p)
        return density_uniform(p, 0.5)
    raise KeyError(name)


def random_problem(nx: int, ny: int, nz: int, seed: int, bc: int = BC_CANTILEVER,
                   rmin: float = 1.5, lo: float = 0.05, hi: float = 1.0):
    """Small ragged test problems: (Problem, rho) with rho ~ U(lo, hi)."""
    p = Problem(f"rand_{nx}x{ny}x{nz}_s{seed}", nx, ny, nz, bc=bc, rmin=rmin)
    rng = np.random.default_rng(seed)
    return p, rng.uniform(lo, hi, p.n_elem)


def random_vector(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)
