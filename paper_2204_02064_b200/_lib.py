"""ctypes binding of libperks_stencil.so (include/perks/perks_stencil.h).

Argument marshalling only: every step of the stencil runs in the CUDA library.  If the shared
library is missing this module raises at import (no CPU fallback exists).
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# PERKS_LIB_PATH overrides the library (development sweeps of compile-time tile parameters only)
LIB_PATH = os.environ.get("PERKS_LIB_PATH") or os.path.join(_PKG, "libperks_stencil.so")

PERKS_OK = 0
STATUS_NAMES = {
    0: "PERKS_OK", 1: "PERKS_ERR_INVALID_ARGUMENT", 2: "PERKS_ERR_INVALID_DOMAIN",
    3: "PERKS_ERR_UNSUPPORTED", 4: "PERKS_ERR_ALIAS", 5: "PERKS_ERR_WORKSPACE",
    6: "PERKS_ERR_NOT_CORESIDENT", 7: "PERKS_ERR_CUDA", 8: "PERKS_ERR_COMM", 9: "PERKS_ERR_OOM",
}
F32, F64 = 0, 1
BC_FRAME, BC_PERIODIC = 0, 1
DIST_BLOB_BYTES = 128  # PERKS_DIST_BLOB_BYTES
VARIANTS = {"auto": 0, "hostloop": 1, "persistent": 2, "perks": 3}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}


class Desc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("extent", ctypes.c_int64 * 3),
        ("npoints", ctypes.c_int32),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("weights", ctypes.POINTER(ctypes.c_double)),
        ("dtype", ctypes.c_int),
        ("bc", ctypes.c_int),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("ctas_per_sm", ctypes.c_int32),
        ("tile", ctypes.c_int32 * 3),
        ("regs_per_thread", ctypes.c_int32),
        ("smem_per_cta", ctypes.c_int32),
        ("cached_cells_reg", ctypes.c_int64),
        ("cached_cells_smem", ctypes.c_int64),
        ("total_cells", ctypes.c_int64),
        ("dram_bytes_per_step", ctypes.c_double),
        ("halo_bytes_per_step", ctypes.c_double),
        ("workspace_bytes", ctypes.c_size_t),
        ("kernel_name", ctypes.c_char * 64),
        ("cached_cells_tmem", ctypes.c_int64),
        ("tmem_cols_per_cta", ctypes.c_int32),
    ]


class CsrDesc(ctypes.Structure):  # perks_csr_desc (include/perks/perks_cg.h)
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_offsets", ctypes.POINTER(ctypes.c_int64)),
        ("col_indices", ctypes.POINTER(ctypes.c_int32)),
        ("values", ctypes.POINTER(ctypes.c_double)),
        ("dtype", ctypes.c_int),
    ]


class CgInfo(ctypes.Structure):  # perks_cg_info
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("items_per_thread", ctypes.c_int32),
        ("tiles", ctypes.c_int32),
        ("smem_per_cta", ctypes.c_int32),
        ("regs_per_thread", ctypes.c_int32),
        ("cached_nnz_smem", ctypes.c_int64),
        ("cached_rows_smem", ctypes.c_int64),
        ("n_rows", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("dram_bytes_per_iter", ctypes.c_double),
        ("unfused_bytes_per_iter", ctypes.c_double),
        ("workspace_bytes", ctypes.c_size_t),
        ("kernel_name", ctypes.c_char * 64),
        ("cached_nnz_tmem", ctypes.c_int64),
        ("tmem_tiles_per_cta", ctypes.c_int32),
        ("smem_tiles_per_cta", ctypes.c_int32),
    ]


CG_POLICIES = {"auto": 0, "imp": 1, "vec": 2, "mat": 3, "mix": 4}
CG_POLICY_NAMES = {v: k for k, v in CG_POLICIES.items()}

# Every symbol include/perks/perks_stencil.h and perks_cg.h declare, with (restype, argtypes).
_VP = ctypes.c_void_p
SIGNATURES = {
    "perks_stencil_create": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.c_int, ctypes.POINTER(_VP)]),
    "perks_stencil_workspace_bytes": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "perks_stencil_run": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP, ctypes.c_size_t,
                                         ctypes.c_int64, _VP]),
    "perks_stencil_run_host": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, ctypes.c_int64]),
    "perks_stencil_query": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(PlanInfo)]),
    "perks_stencil_launch_count": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int64,
                                                  ctypes.POINTER(ctypes.c_int64)]),
    "perks_stencil_create_dist": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, ctypes.POINTER(_VP)]),
    "perks_stencil_dist_export": (ctypes.c_int, [_VP, _VP]),
    "perks_stencil_dist_connect": (ctypes.c_int, [_VP, _VP, _VP]),
    "perks_stencil_run_group": (ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, ctypes.c_int,
                                               ctypes.POINTER(_VP), ctypes.POINTER(_VP),
                                               ctypes.POINTER(_VP), ctypes.POINTER(ctypes.c_size_t),
                                               ctypes.c_int64, _VP]),
    "perks_stencil_destroy": (ctypes.c_int, [_VP]),
    "perks_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "perks_last_cuda_error": (ctypes.c_int, []),
    "perks_version": (ctypes.c_char_p, []),
    # include/perks/perks_cg.h
    "perks_cg_create": (ctypes.c_int, [ctypes.POINTER(CsrDesc), ctypes.c_int, ctypes.POINTER(_VP)]),
    "perks_cg_workspace_bytes": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_size_t)]),
    "perks_cg_spmv": (ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_size_t, _VP]),
    "perks_cg_solve": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, _VP, _VP, ctypes.c_int64,
                                      ctypes.c_double, _VP, _VP, _VP, ctypes.c_size_t, _VP]),
    "perks_cg_solve_host": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, _VP, _VP, ctypes.c_int64,
                                           ctypes.c_double, _VP, _VP]),
    "perks_cg_query": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.POINTER(CgInfo)]),
    "perks_cg_partition": (ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]),
    "perks_cg_destroy": (ctypes.c_int, [_VP]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class PerksError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        name = STATUS_NAMES.get(status, str(status))
        cuda = lib.perks_last_cuda_error() if status == 7 else 0
        super().__init__(f"{what}: {name}" + (f" (cudaError {cuda})" if cuda else ""))
        self.status = status
        self.name = name


def check(status: int, what: str = "") -> None:
    if status != PERKS_OK:
        raise PerksError(status, what)
