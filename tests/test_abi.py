"""C-ABI library: loads, exports every symbol include/tomo.h declares, and its host-only
tables (KE, load list, filter taps, sizes, argument validation) match the oracle
bit-exactly / to rounding. No CUDA call is made here (CPU-only container)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from oracle import fem, filt, grid
from paper_2104_12282_b200 import build as tbuild
from paper_2104_12282_b200 import tomo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    tbuild.build()
    return tomo.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "tomo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tomo_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(tomo.EXPORTS) == names  # the binding covers the whole header


def _create(lib, nx, ny, nz, bc=1, rmin=1.5, nu=0.3, h=1.0, E0=1.0, Emin=1e-9, penal=3.0,
            fixed=(), ldofs=(), lvals=(), load_total=-1.0):
    g = tomo._Grid(nx, ny, nz, h)
    fa = (C.c_int64 * max(1, len(fixed)))(*fixed)
    la = (C.c_int64 * max(1, len(ldofs)))(*ldofs)
    va = (C.c_double * max(1, len(lvals)))(*lvals)
    b = tomo._BC(bc, load_total, fa, len(fixed), la, va, len(ldofs))
    hnd = C.c_void_p()
    rc = lib.tomo_create(C.byref(hnd), C.byref(g), E0, Emin, nu, penal, rmin, C.byref(b))
    return rc, hnd


def test_ke_matches_oracle_quadrature(lib):
    for nu, h in [(0.3, 1.0), (0.25, 2.0), (0.45, 0.5)]:
        rc, hnd = _create(lib, 2, 2, 2, nu=nu, h=h)
        assert rc == 0
        buf = (C.c_double * 576)()
        assert lib.tomo_get_ke(hnd, buf) == 0
        KE = np.array(buf[:]).reshape(24, 24)
        ref = fem.element_stiffness(nu, h)
        assert np.max(np.abs(KE - ref)) <= 1e-15 * np.max(np.abs(ref)) * 10
        lib.tomo_destroy(hnd)


@pytest.mark.parametrize("dims,bc", [((24, 12, 12), 1), ((5, 3, 7), 1), ((1, 1, 1), 1),
                                     ((96, 32, 32), 2), ((3, 4, 2), 2)])
def test_loads_bit_exact(lib, dims, bc):
    rc, hnd = _create(lib, *dims, bc=bc)
    assert rc == 0
    n = C.c_int64(0)
    assert lib.tomo_get_load(hnd, None, None, C.byref(n)) == 0
    d = (C.c_int64 * n.value)()
    v = (C.c_double * n.value)()
    assert lib.tomo_get_load(hnd, d, v, C.byref(n)) == 0
    fixed, odofs, ovals = grid.bc_for(bc, *dims)
    assert list(d) == odofs.tolist()
    assert np.array_equal(np.array(v[:]), ovals)  # bit-exact: same single division
    sz = (C.c_int64 * 5)()
    lib.tomo_sizes(hnd, sz)
    assert tuple(sz[:3]) == grid.counts(*dims)
    lib.tomo_destroy(hnd)


@pytest.mark.parametrize("rmin,ntaps", [(1.5, 19), (2.0, 27), (3.0, 93), (0.9, 1), (7.2, 1551)])
def test_filter_taps_bit_exact(lib, rmin, ntaps):
    rc, hnd = _create(lib, 4, 4, 4, rmin=rmin)
    assert rc == 0
    n = C.c_int(0)
    assert lib.tomo_get_filter_taps(hnd, None, None, C.byref(n)) == 0
    assert n.value == ntaps
    o = (C.c_int * (3 * n.value))()
    w = (C.c_double * n.value)()
    assert lib.tomo_get_filter_taps(hnd, o, w, C.byref(n)) == 0
    ref = filt.taps(rmin)
    assert [tuple(o[3 * i:3 * i + 3]) for i in range(n.value)] == [t[:3] for t in ref]
    assert np.array_equal(np.array(w[:]), np.array([t[3] for t in ref]))
    lib.tomo_destroy(hnd)


@pytest.mark.parametrize("kw,why", [
    (dict(nx=0, ny=1, nz=1), "nel"), (dict(nx=1, ny=1, nz=1, nu=0.5), "nu"),
    (dict(nx=1, ny=1, nz=1, Emin=0.0), "Emin"), (dict(nx=1, ny=1, nz=1, penal=0.5), "penal"),
    (dict(nx=1, ny=1, nz=1, rmin=0.0), "rmin"), (dict(nx=1, ny=1, nz=1, h=-1.0), "h"),
    (dict(nx=1, ny=1, nz=1, bc=3, fixed=(2,), ldofs=(2,), lvals=(1.0,)), "load on fixed"),
    (dict(nx=1, ny=1, nz=1, bc=3, fixed=(24,)), "range"), (dict(nx=1, ny=1, nz=1, bc=9), "kind"),
    (dict(nx=1024, ny=1024, nz=1024), "32-bit internal DOF index"),
])
def test_create_validation(lib, kw, why):
    nx, ny, nz = kw.pop("nx"), kw.pop("ny"), kw.pop("nz")
    rc, hnd = _create(lib, nx, ny, nz, **kw)
    assert rc == tomo.TomoError(-1, "").code == -1, why
    msg = lib.tomo_last_error(hnd)
    assert msg and len(msg) > 3
    lib.tomo_destroy(hnd)


def test_unbound_calls_report_no_workspace(lib):
    rc, hnd = _create(lib, 2, 2, 2)
    assert rc == 0
    assert lib.tomo_workspace_bytes(hnd) > 0
    c = C.c_double()
    assert lib.tomo_compliance(hnd, None, 81, C.byref(c)) == -9  # TOMO_ENOWORKSPACE
    lib.tomo_destroy(hnd)


def test_explicit_bc_merges_duplicate_loads(lib):
    rc, hnd = _create(lib, 1, 1, 1, bc=3, fixed=(0, 1, 2), ldofs=(5, 5, 8), lvals=(1.0, 2.0, -1.0))
    assert rc == 0
    n = C.c_int64(4)
    d = (C.c_int64 * 4)()
    v = (C.c_double * 4)()
    assert lib.tomo_get_load(hnd, d, v, C.byref(n)) == 0
    assert n.value == 2 and list(d[:2]) == [5, 8] and list(v[:2]) == [3.0, -1.0]
    lib.tomo_destroy(hnd)


def test_largest_grid_under_the_index_limit_is_accepted(lib):
    """The maximum size: the internal (padded) DOF index is 32-bit, so the largest accepted
    grid has 3 nnx_pad (ny+1) (nz+1) < 2^31 - 64 (890^3: 2.1e9 DOFs); its workspace still
    fits a B200's HBM (183,359 MiB per nvidia-smi)."""
    rc, hnd = _create(lib, 890, 890, 890)
    assert rc == 0
    assert lib.tomo_workspace_bytes(hnd) < 183359 * 1024 ** 2
    lib.tomo_destroy(hnd)
    rc, hnd = _create(lib, 900, 900, 900)
    assert rc == -1
    lib.tomo_destroy(hnd)


def test_workspace_fits_hbm_at_largest_config(lib):
    rc, hnd = _create(lib, 256, 128, 128)
    assert rc == 0
    assert lib.tomo_workspace_bytes(hnd) < 2 * 1024 ** 3  # < 2 GB of 180 GB HBM
    lib.tomo_destroy(hnd)


@pytest.mark.parametrize("dims,bc,nb", [((8, 4, 4), 1, 2), ((24, 12, 12), 1, 4), ((12, 8, 8), 2, 2),
                                        ((6, 3, 3), 1, 3), ((5, 3, 7), 1, 1)])
def test_coarse_context_loads_match_oracle_restriction(lib, dims, bc, nb):
    """tomo_create_coarse (host-only) vs oracle.twoscale.restrict_bc: load DOFs bit-exact,
    values to rounding, sizes by the SPEC.md l.386 rule."""
    from oracle import twoscale
    rc, fine = _create(lib, *dims, bc=bc)
    assert rc == 0
    coarse = C.c_void_p()
    assert lib.tomo_create_coarse(C.byref(coarse), fine, nb) == 0
    sz = (C.c_int64 * 5)()
    lib.tomo_sizes(coarse, sz)
    assert tuple(sz[:3]) == grid.counts(*(d // nb for d in dims))
    n = C.c_int64(0)
    lib.tomo_get_load(coarse, None, None, C.byref(n))
    d = (C.c_int64 * max(1, n.value))()
    v = (C.c_double * max(1, n.value))()
    lib.tomo_get_load(coarse, d, v, C.byref(n))
    fixed, ld, lv = grid.bc_for(bc, *dims)
    fc, ldc, lvc = twoscale.restrict_bc(*dims, nb, fixed, ld, lv)
    order = np.argsort(np.array(d[:n.value]))
    assert np.array_equal(np.array(d[:n.value])[order], ldc)
    assert np.allclose(np.array(v[:n.value])[order], lvc, rtol=1e-15, atol=0)
    bad = C.c_void_p()
    assert lib.tomo_create_coarse(C.byref(bad), fine, 7) == -1  # 7 divides none of the grids
    lib.tomo_destroy(coarse)
    lib.tomo_destroy(fine)


def test_concurrent_create_is_thread_safe(lib):
    """tomo_create from many threads at once (ctypes releases the GIL): every context gets its
    own KE and passes its Walsh-pattern self-check (the basis-change scratch was a
    shared static array)."""
    import threading
    nus = [0.05 + 0.4 * i / 63 for i in range(64)]
    res = [None] * len(nus)

    def work(i):
        rc, hnd = _create(lib, 3, 2, 2, nu=nus[i])
        buf = (C.c_double * 576)()
        ok = rc == 0 and lib.tomo_get_ke(hnd, buf) == 0
        res[i] = (ok, np.array(buf[:]).reshape(24, 24))
        lib.tomo_destroy(hnd)

    for _ in range(3):
        th = [threading.Thread(target=work, args=(i,)) for i in range(len(nus))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for i, nu in enumerate(nus):
            ok, KE = res[i]
            assert ok, nu
            ref = fem.element_stiffness(nu, 1.0)
            assert np.max(np.abs(KE - ref)) <= 1e-14 * np.max(np.abs(ref))
