"""C-ABI checks that need no GPU: the library loads, exports every symbol the public header
declares, and rejects bad descriptors before touching CUDA (include/perks/perks_stencil.h)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "perks", "perks_stencil.h")
HEADERS = [HEADER, os.path.join(ROOT, "include", "perks", "perks_cg.h")]


def _declared_symbols():
    out = set()
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        out |= set(re.findall(r"\b(perks_[a-z_]+)\s*\(", src))
    return sorted(out)


def test_library_exports_every_declared_symbol():
    from paper_2204_02064_b200 import _lib
    syms = _declared_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(_lib.lib, s), s
        assert s in _lib.SIGNATURES, f"binding lacks {s}"


def test_status_strings_and_version():
    from paper_2204_02064_b200 import _lib
    for code, name in _lib.STATUS_NAMES.items():
        assert _lib.lib.perks_status_string(code).decode() == name
    assert b"sm_100a" in _lib.lib.perks_version()


def _create(ndim, ext, offs, w, dtype=0, bc=0):
    from paper_2204_02064_b200 import _lib
    offs = np.ascontiguousarray(np.asarray(offs, dtype=np.int32).reshape(-1, 3))
    w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
    d = _lib.Desc()
    d.ndim = ndim
    d.extent[:] = ext
    d.npoints = offs.shape[0]
    d.offsets = offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    d.dtype = dtype
    d.bc = bc
    h = ctypes.c_void_p()
    st = _lib.lib.perks_stencil_create(ctypes.byref(d), 0, ctypes.byref(h))
    if st == 0:
        _lib.lib.perks_stencil_destroy(h)
    return _lib.STATUS_NAMES[st]


def test_create_validation_without_gpu():
    import seeded_inputs as si
    o5, w5 = si.preset("2d5pt")
    o7, w7 = si.preset("3d7pt")
    assert _create(4, (8, 8, 1), o5, w5) == "PERKS_ERR_INVALID_ARGUMENT"       # bad ndim
    assert _create(2, (8, 8, 2), o5, w5) == "PERKS_ERR_INVALID_DOMAIN"         # nz != 1 in 2D
    assert _create(2, (2, 8, 1), o5, w5) == "PERKS_ERR_INVALID_DOMAIN"         # nx < 2r+1
    assert _create(3, (8, 8, 2), o7, w7) == "PERKS_ERR_INVALID_DOMAIN"         # nz < 2r+1
    assert _create(2, (8, 8, 1), o7, w7) == "PERKS_ERR_INVALID_ARGUMENT"       # dz in 2D
    assert _create(2, (8, 8, 1), o5, w5, dtype=7) == "PERKS_ERR_INVALID_ARGUMENT"
    assert _create(2, (8, 8, 1), o5, [1.0, float("nan"), 0, 0, 0]) == "PERKS_ERR_INVALID_ARGUMENT"
    # point sets without a specialised kernel run on the general kernels up to radius 6 (2D,
    # k2d_wide.cu) / 3 (3D, k3d_wide.cu); beyond that they are unsupported
    assert _create(3, (12, 12, 12), [(0, 0, 4), (0, 0, 0)], [0.5, 0.5]) == "PERKS_ERR_UNSUPPORTED"  # 3D r = 4
    assert _create(2, (20, 20, 1), [(7, 0, 0), (0, 0, 0)], [0.5, 0.5]) == "PERKS_ERR_UNSUPPORTED"  # r = 7
    # PERIODIC runs on the general kernels (single GPU): the same radius limits apply
    assert _create(2, (20, 20, 1), [(7, 0, 0), (0, 0, 0)], [0.5, 0.5], bc=1) == "PERKS_ERR_UNSUPPORTED"
    assert _create(3, (12, 12, 12), [(0, 0, 4), (0, 0, 0)], [0.5, 0.5], bc=1) == "PERKS_ERR_UNSUPPORTED"
    assert _create(2, (8, 8, 1), o5, w5, bc=2) == "PERKS_ERR_INVALID_ARGUMENT"  # unknown bc


def test_periodic_slabs_unsupported_without_gpu():
    import seeded_inputs as si
    from paper_2204_02064_b200 import _lib
    o7, w7 = si.preset("3d7pt")
    offs = np.ascontiguousarray(np.asarray(o7, dtype=np.int32).reshape(-1, 3))
    w = np.ascontiguousarray(np.asarray(w7, dtype=np.float64))
    d = _lib.Desc()
    d.ndim = 3
    d.extent[:] = (16, 16, 8)
    d.npoints = offs.shape[0]
    d.offsets = offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    d.weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    d.dtype = 0
    d.bc = 1
    h = ctypes.c_void_p()
    st = _lib.lib.perks_stencil_create_dist(ctypes.byref(d), 0, 0, 2, ctypes.byref(h))
    assert _lib.STATUS_NAMES[st] == "PERKS_ERR_UNSUPPORTED"


def test_null_arguments():
    from paper_2204_02064_b200 import _lib
    L = _lib.lib
    assert L.perks_stencil_create(None, 0, None) == 1
    assert L.perks_stencil_run(None, 0, None, None, None, 0, 1, None) == 1
    assert L.perks_stencil_destroy(None) == 1
