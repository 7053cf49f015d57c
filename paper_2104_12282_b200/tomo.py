"""Thin ctypes binding of libtomo (include/tomo.h): argument marshalling only.

Every step of the exact-gradient path runs in libtomo's CUDA kernels; torch supplies device
memory (tensors, the workspace) and the stream. There is no CPU fallback: if the library
is missing or no GPU is present, constructing :class:`Tomo` raises.

Names follow the C ABI: ``apply`` (K_hat u), ``solve`` (Jacobi-PCG, PAPER.md
l.184/240), ``compliance`` (Eq. 4), ``sensitivity`` (Eq. 5), ``filter`` (P / P^T, PAPER.md
l.180/184), ``volume_grad`` (P^T v), ``oc_update`` (OC), ``evaluate`` (one
exact-gradient evaluation).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOMO_LIB_PATH") or os.path.join(_PKG, "lib", "libtomo.so")

TOMO_BC_CANTILEVER = 1
TOMO_BC_MBB_HALF = 2
TOMO_BC_EXPLICIT = 3

STATUS = {0: "TOMO_OK", -1: "TOMO_EINVAL", -2: "TOMO_EDOMAIN", -3: "TOMO_ESIZE",
          -4: "TOMO_EBREAKDOWN", -5: "TOMO_EPRECOND", -6: "TOMO_ENAN", -7: "TOMO_EBRACKET",
          -8: "TOMO_ECUDA", -9: "TOMO_ENOWORKSPACE"}


class TomoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class _Grid(C.Structure):
    _fields_ = [("nelx", C.c_int), ("nely", C.c_int), ("nelz", C.c_int), ("h", C.c_double)]


class _BC(C.Structure):
    _fields_ = [("kind", C.c_int), ("load_total", C.c_double),
                ("fixed_dofs", C.POINTER(C.c_int64)), ("n_fixed", C.c_int64),
                ("load_dofs", C.POINTER(C.c_int64)), ("load_vals", C.POINTER(C.c_double)),
                ("n_loads", C.c_int64)]


class SolveInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("rel_res_recursive", C.c_double), ("rel_res_true", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None

# (name, restype, argtypes)
_SIGS = [
    ("tomo_create", C.c_int, [C.POINTER(C.c_void_p), C.POINTER(_Grid), C.c_double, C.c_double,
                              C.c_double, C.c_double, C.c_double, C.POINTER(_BC)]),
    ("tomo_workspace_bytes", C.c_size_t, [C.c_void_p]),
    ("tomo_bind", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    ("tomo_destroy", None, [C.c_void_p]),
    ("tomo_last_error", C.c_char_p, [C.c_void_p]),
    ("tomo_sizes", C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    ("tomo_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64]),
    ("tomo_solve", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_double,
                             C.c_int, C.POINTER(SolveInfo)]),
    ("tomo_compliance", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double)]),
    ("tomo_sensitivity", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_double)]),
    ("tomo_filter", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int]),
    ("tomo_volume_grad", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    ("tomo_oc_update", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                 C.c_double, C.c_double, C.c_double, C.c_void_p,
                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    ("tomo_evaluate", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(SolveInfo)]),
    ("tomo_evaluate_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                     C.c_int, C.POINTER(C.c_double), C.POINTER(SolveInfo)]),
    ("tomo_get_ke", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("tomo_get_fixed_mask", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tomo_get_load", C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                C.POINTER(C.c_int64)]),
    ("tomo_get_filter_taps", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int)]),
    ("tomo_get_element_dofs", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tomo_get_neighbor_counts", C.c_int, [C.c_void_p, C.c_void_p]),
    ("tomo_get_jacobi", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tomo_launch_count", C.c_int64, [C.c_void_p]),
    ("tomo_bench_dfma", C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("tomo_set_profiling", C.c_int, [C.c_void_p, C.c_int]),
    ("tomo_set_graph", C.c_int, [C.c_void_p, C.c_int]),
    ("tomo_set_pcg_exact_beta", C.c_int, [C.c_void_p, C.c_int]),
    ("tomo_set_history", C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    ("tomo_profile_times", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("tomo_bench_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    ("tomo_create_coarse", C.c_int, [C.POINTER(C.c_void_p), C.c_void_p, C.c_int]),
    ("tomo_coarsen", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64]),
    ("tomo_mg_workspace_bytes", C.c_size_t, [C.c_void_p, C.c_int]),
    ("tomo_mg_bind", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t]),
    ("tomo_mg_params", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double]),
    ("tomo_solve_mg", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_double,
                                C.c_int, C.POINTER(SolveInfo)]),
]
EXPORTS = [s[0] for s in _SIGS]


def load_library(path: str = LIB_PATH):
    """Load libtomo.so (no CUDA call is made). Raises if the built library is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libtomo not built: {path} missing (run python -m "
                               "paper_2104_12282_b200.build); there is no CPU fallback")
        lib = C.CDLL(path)
        for name, res, args in _SIGS:
            if os.environ.get("TOMO_LIB_PATH") and not hasattr(lib, name):
                continue  # A/B timing of a variant build (scripts/build_variants.py)
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class _DeviceLib:
    """libtomo calls made with this context's device current: the library launches on the
    current device and reads its SM count from it (a context on cuda:1 must not run while
    cuda:0 is current)."""

    def __init__(self, lib, device: torch.device):
        self._lib, self._dev = lib, device

    def __getattr__(self, name):
        fn = getattr(self._lib, name)

        def call(*args):
            with torch.cuda.device(self._dev):
                return fn(*args)
        return call


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _f64(t: torch.Tensor, n: int, name: str):
    if t.dtype != torch.float64 or t.numel() != n:
        raise ValueError(f"{name}: expected float64 tensor of {n} elements, got {t.dtype} {t.numel()}")
    return t


@dataclass
class Params:
    nelx: int
    nely: int
    nelz: int
    E0: float = 1.0
    Emin: float = 1e-9
    nu: float = 0.3
    penal: float = 3.0
    rmin: float = 1.5
    h: float = 1.0
    bc: int = TOMO_BC_CANTILEVER
    load_total: float = -1.0
    fixed_dofs: tuple = ()
    load_dofs: tuple = ()
    load_vals: tuple = ()


class Tomo:
    """One problem context bound to a torch-allocated workspace on the current device/stream."""

    def __init__(self, p: Params, device: str | torch.device = "cuda", stream=None, _handle=None):
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("libtomo needs a CUDA device (no CPU fallback)")
        self.p = p
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.lib = _DeviceLib(lib, self.device)
        if _handle is not None:  # context already created (tomo_create_coarse)
            self._bind(_handle, stream)
            return
        g = _Grid(p.nelx, p.nely, p.nelz, p.h)
        fixed = (C.c_int64 * max(1, len(p.fixed_dofs)))(*p.fixed_dofs)
        ldofs = (C.c_int64 * max(1, len(p.load_dofs)))(*p.load_dofs)
        lvals = (C.c_double * max(1, len(p.load_vals)))(*p.load_vals)
        bc = _BC(p.bc, p.load_total, fixed, len(p.fixed_dofs), ldofs, lvals, len(p.load_dofs))
        self._keep = (fixed, ldofs, lvals)
        h = C.c_void_p()
        lib = self.lib
        rc = lib.tomo_create(C.byref(h), C.byref(g), p.E0, p.Emin, p.nu, p.penal, p.rmin, C.byref(bc))
        self.h = h
        if rc != 0:
            msg = lib.tomo_last_error(h).decode() if h.value else "tomo_create failed"
            if h.value:
                lib.tomo_destroy(h)
                self.h = C.c_void_p()
            raise TomoError(rc, msg)
        self._bind(h, stream)

    def _bind(self, h, stream):
        lib = self.lib
        self.h = h
        sz = (C.c_int64 * 5)()
        lib.tomo_sizes(h, sz)
        self.n_e, self.n_n, self.n_dof, self.n_loads, self.n_taps = (int(v) for v in sz)
        nbytes = lib.tomo_workspace_bytes(h)
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        # device buffers are allocated on the bound stream (the caching allocator then never
        # hands them to another stream while the library may still use them)
        with torch.cuda.stream(self.stream):
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self._check(lib.tomo_bind(h, C.c_void_p(base + off), nbytes, C.c_void_p(self.stream.cuda_stream)))

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc: int) -> int:
        if rc < 0:
            raise TomoError(rc, self.lib.tomo_last_error(self.h).decode())
        return rc

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.tomo_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def zeros_dof(self):
        # allocated and zeroed on the bound stream, where the library will read it
        with torch.cuda.stream(self.stream):
            return torch.zeros(self.n_dof, dtype=torch.float64, device=self.device)

    def zeros_elem(self):
        with torch.cuda.stream(self.stream):
            return torch.zeros(self.n_e, dtype=torch.float64, device=self.device)

    @property
    def launches(self) -> int:
        return int(self.lib.tomo_launch_count(self.h))

    # ------------------------------------------------------------------ the path
    def apply(self, rho: torch.Tensor, u: torch.Tensor, y: torch.Tensor | None = None):
        y = self.zeros_dof() if y is None else y
        self._check(self.lib.tomo_apply(self.h, _ptr(_f64(rho, self.n_e, "rho")), self.n_e,
                                        _ptr(_f64(u, self.n_dof, "u")), _ptr(_f64(y, self.n_dof, "y")),
                                        self.n_dof))
        return y

    def solve(self, rho: torch.Tensor, u: torch.Tensor | None = None, tol: float = 1e-10,
              max_iters: int = 50000):
        u = self.zeros_dof() if u is None else u
        info = SolveInfo()
        self._check(self.lib.tomo_solve(self.h, _ptr(_f64(rho, self.n_e, "rho")), self.n_e,
                                        _ptr(_f64(u, self.n_dof, "u")), self.n_dof, tol, max_iters,
                                        C.byref(info)))
        return u, info

    def compliance(self, u: torch.Tensor) -> float:
        c = C.c_double()
        self._check(self.lib.tomo_compliance(self.h, _ptr(_f64(u, self.n_dof, "u")), self.n_dof, C.byref(c)))
        return c.value

    def sensitivity(self, rho, u, dc=None, ce=None, energy: bool = False):
        dc = self.zeros_elem() if dc is None else dc
        en = C.c_double()
        self._check(self.lib.tomo_sensitivity(self.h, _ptr(_f64(rho, self.n_e, "rho")),
                                              _ptr(_f64(u, self.n_dof, "u")), _ptr(_f64(dc, self.n_e, "dc")),
                                              _ptr(ce), C.byref(en) if energy else None))
        return (dc, en.value) if energy else dc

    def filter(self, x: torch.Tensor, out: torch.Tensor | None = None, transpose: bool = False):
        out = self.zeros_elem() if out is None else out
        self._check(self.lib.tomo_filter(self.h, _ptr(_f64(x, self.n_e, "in")), _ptr(_f64(out, self.n_e, "out")),
                                         self.n_e, 1 if transpose else 0))
        return out

    def volume_grad(self, out: torch.Tensor | None = None):
        out = self.zeros_elem() if out is None else out
        self._check(self.lib.tomo_volume_grad(self.h, _ptr(_f64(out, self.n_e, "dv")), self.n_e))
        return out

    def oc_update(self, x, g, dv, volfrac, move=0.2, eta=0.5, out=None):
        out = self.zeros_elem() if out is None else out
        lam = C.c_double()
        steps = C.c_int()
        self._check(self.lib.tomo_oc_update(self.h, _ptr(_f64(x, self.n_e, "x")), _ptr(_f64(g, self.n_e, "g")),
                                            _ptr(_f64(dv, self.n_e, "dv")), self.n_e, volfrac, move, eta,
                                            _ptr(_f64(out, self.n_e, "xnew")), C.byref(lam), C.byref(steps)))
        return out, lam.value, steps.value

    def evaluate(self, rho, u=None, dc=None, dcf=None, tol=1e-10, max_iters=50000):
        """One exact-gradient evaluation: (u, c, dcf, info)."""
        u = self.zeros_dof() if u is None else u
        dcf = self.zeros_elem() if dcf is None else dcf
        c = C.c_double()
        info = SolveInfo()
        self._check(self.lib.tomo_evaluate(self.h, _ptr(_f64(rho, self.n_e, "rho")), _ptr(_f64(u, self.n_dof, "u")),
                                           _ptr(dc), _ptr(_f64(dcf, self.n_e, "dcf")), tol, max_iters,
                                           C.byref(c), C.byref(info)))
        return u, c.value, dcf, info

    def evaluate_host(self, rho_h: torch.Tensor, dcf_h: torch.Tensor, u_h: torch.Tensor | None = None,
                      tol=1e-10, max_iters=50000):
        """Same with host (ideally pinned) CPU tensors; copies happen inside the C call."""
        for t in (rho_h, dcf_h) + ((u_h,) if u_h is not None else ()):
            if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
                raise ValueError("evaluate_host takes contiguous float64 CPU tensors")
        c = C.c_double()
        info = SolveInfo()
        self._check(self.lib.tomo_evaluate_host(self.h, C.c_void_p(rho_h.data_ptr()),
                                                C.c_void_p(u_h.data_ptr()) if u_h is not None else None,
                                                C.c_void_p(dcf_h.data_ptr()), tol, max_iters,
                                                C.byref(c), C.byref(info)))
        return c.value, info

    # ------------------------------------------------------------------ two-scale coarse path
    def coarse(self, nb: int) -> "Tomo":
        """Context of the coarse problem K_C(z_C) u_C = f_C (tomo_create_coarse)."""
        h = C.c_void_p()
        rc = self.lib.tomo_create_coarse(C.byref(h), self.h, nb)
        if rc != 0:
            if h.value:
                self.lib.tomo_destroy(h)
            raise TomoError(rc, "tomo_create_coarse failed (nb must divide the grid)")
        p = self.p
        cp = Params(p.nelx // nb, p.nely // nb, p.nelz // nb, E0=p.E0, Emin=p.Emin, nu=p.nu,
                    penal=p.penal, rmin=p.rmin, h=p.h * nb, bc=TOMO_BC_EXPLICIT)
        return Tomo(cp, device=self.device, stream=self.stream, _handle=h)

    def coarsen(self, z: torch.Tensor, nb: int, out: torch.Tensor | None = None):
        n_ec = (self.p.nelx // nb) * (self.p.nely // nb) * (self.p.nelz // nb)
        with torch.cuda.stream(self.stream):
            out = torch.zeros(n_ec, dtype=torch.float64, device=self.device) if out is None else out
        self._check(self.lib.tomo_coarsen(self.h, _ptr(_f64(z, self.n_e, "z")), nb,
                                          _ptr(_f64(out, n_ec, "zc")), n_ec))
        return out

    # ------------------------------------------------------------------ multigrid
    def mg_setup(self, levels: int, nu: int = 2, omega: float = 0.3, coarse_iters: int = 30,
                 coarse_tol: float = 1e-2):
        nbytes = self.lib.tomo_mg_workspace_bytes(self.h, levels)
        if not nbytes:
            raise TomoError(-1, f"{levels} MG levels impossible on this grid")
        with torch.cuda.stream(self.stream):
            self.mg_workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.mg_workspace.data_ptr()
        self._check(self.lib.tomo_mg_bind(self.h, levels, C.c_void_p(base + (-base) % 256), nbytes))
        self._check(self.lib.tomo_mg_params(self.h, nu, omega, coarse_iters, coarse_tol))

    def solve_mg(self, rho: torch.Tensor, u: torch.Tensor | None = None, tol: float = 1e-10,
                 max_iters: int = 2000):
        u = self.zeros_dof() if u is None else u
        info = SolveInfo()
        self._check(self.lib.tomo_solve_mg(self.h, _ptr(_f64(rho, self.n_e, "rho")), self.n_e,
                                           _ptr(_f64(u, self.n_dof, "u")), self.n_dof, tol, max_iters,
                                           C.byref(info)))
        return u, info

    # ------------------------------------------------------------------ introspection
    def ke(self):
        buf = (C.c_double * 576)()
        self._check(self.lib.tomo_get_ke(self.h, buf))
        return torch.tensor(list(buf), dtype=torch.float64).reshape(24, 24)

    def fixed_mask(self):
        with torch.cuda.stream(self.stream):
            m = torch.zeros(self.n_dof, dtype=torch.uint8, device=self.device)
        self._check(self.lib.tomo_get_fixed_mask(self.h, _ptr(m)))
        return m

    def loads(self):
        n = C.c_int64(self.n_loads)
        d = (C.c_int64 * max(1, self.n_loads))()
        v = (C.c_double * max(1, self.n_loads))()
        self._check(self.lib.tomo_get_load(self.h, d, v, C.byref(n)))
        return list(d)[: n.value], list(v)[: n.value]

    def filter_taps(self):
        n = C.c_int(self.n_taps)
        o = (C.c_int * max(3, 3 * self.n_taps))()
        w = (C.c_double * max(1, self.n_taps))()
        self._check(self.lib.tomo_get_filter_taps(self.h, o, w, C.byref(n)))
        return [tuple(o[3 * i:3 * i + 3]) for i in range(n.value)], list(w)[: n.value]

    def element_dofs(self):
        with torch.cuda.stream(self.stream):
            m = torch.empty(self.n_e * 24, dtype=torch.int64, device=self.device)
        self._check(self.lib.tomo_get_element_dofs(self.h, _ptr(m)))
        return m.view(self.n_e, 24)

    def neighbor_counts(self):
        with torch.cuda.stream(self.stream):
            m = torch.empty(self.n_e, dtype=torch.int32, device=self.device)
        self._check(self.lib.tomo_get_neighbor_counts(self.h, _ptr(m)))
        return m

    def jacobi(self, rho):
        with torch.cuda.stream(self.stream):
            out = torch.empty(self.n_n, dtype=torch.float64, device=self.device)
        self._check(self.lib.tomo_get_jacobi(self.h, _ptr(_f64(rho, self.n_e, "rho")), _ptr(out)))
        return out

    # ------------------------------------------------------------------ measurement helpers
    def bench_dfma(self):
        gf = C.c_double()
        ms = C.c_double()
        self._check(self.lib.tomo_bench_dfma(self.h, C.byref(gf), C.byref(ms)))
        return gf.value, ms.value

    def set_pcg_exact_beta(self, on: bool):
        """Textbook beta from the explicit r_{k+1} (one extra pass per iteration) instead of
        the single-pass prediction (reading R1)."""
        self._check(self.lib.tomo_set_pcg_exact_beta(self.h, 1 if on else 0))

    def set_graph(self, on: bool):
        """PCG loop as one CUDA graph (default) or host-batched launches (ncu-visible)."""
        self._check(self.lib.tomo_set_graph(self.h, 1 if on else 0))

    def set_history(self, n: int):
        """Record r_k^T r_k of every PCG launch of the next solves (n entries, device)."""
        with torch.cuda.stream(self.stream):
            self.hist = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self._check(self.lib.tomo_set_history(self.h, _ptr(self.hist) if n > 0 else None, n))
        return self.hist

    def set_profiling(self, on: bool):
        self._check(self.lib.tomo_set_profiling(self.h, 1 if on else 0))

    def profile_times(self):
        t = (C.c_double * 3)()
        self._check(self.lib.tomo_profile_times(self.h, t))
        return {"k_a_ms": t[0], "k_b_ms": t[1], "n": int(t[2])}

    def bench_apply(self, rho: torch.Tensor, reps: int = 100) -> float:
        ms = C.c_double()
        self._check(self.lib.tomo_bench_apply(self.h, _ptr(_f64(rho, self.n_e, "rho")), reps, C.byref(ms)))
        return ms.value


def params_from_problem(p) -> Params:
    """Map an inputs.Problem (seeded configs) to ABI parameters."""
    return Params(nelx=p.nx, nely=p.ny, nelz=p.nz, E0=p.E0, Emin=p.Emin, nu=p.nu, penal=p.penal,
                  rmin=p.rmin, h=p.h, bc=p.bc, load_total=p.load_total)
