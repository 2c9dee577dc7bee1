"""CPU oracle for the PERKS stencil time loop (arXiv 2204.02064).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2204_02064_b200``) never imports it and
shares no code with it (the oracle is plain C in ``stencil_oracle.c``; this
file only marshals numpy arrays into it).

What it computes: T out-of-place applications of the stencil operator
``x(c)^{k+1} = sum_p w_p x(c+d_p)^k`` (PAPER.md P:182-187 Eq. ``iterative``,
P:204-213 Eq. ``iterativeStencil``), first term a rounded multiply, the rest
fused multiply-adds in list order, in the storage dtype, FRAME or PERIODIC
boundary (DESIGN.md "Readings" R1-R9).

Pins: ``tests/test_oracle_pins.py`` (identity, shift closed form, constant
fixed point, Fourier-mode decay, exact-rational brute force, linearity,
composability, maximum principle).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stencil_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "cg_oracle.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

BC_FRAME = 0
BC_PERIODIC = 1

_ERR = {1: "INVALID_ARGUMENT", 2: "INVALID_DOMAIN", 3: "OOM", 4: "NOT_SPD"}


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code} ({_ERR.get(code, '?')})")
        self.code = code
        self.name = _ERR.get(code, "?")


def build(force: bool = False) -> str:
    """Compile liboracle.so (stencil_oracle.c + cg_oracle.c) with gcc: -O2 -mfma
    -ffp-contract=off (no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(s) for s in _SRCS)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-mfma", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-std=c11", "-shared", "-fPIC", "-o", tmp, *_SRCS, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i64p = ctypes.POINTER(ctypes.c_int64)
            i32p = ctypes.POINTER(ctypes.c_int32)
            for name in ("oracle_stencil_f64", "oracle_stencil_f32"):
                f = getattr(lib, name)
                f.restype = ctypes.c_int
                f.argtypes = [ctypes.c_int, i64p, ctypes.c_int, i32p, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int]
            for name in ("oracle_csr_spmv_f64", "oracle_csr_spmv_f32"):
                f = getattr(lib, name)
                f.restype = ctypes.c_int
                f.argtypes = [ctypes.c_int64, i64p, i32p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_int]
            for name in ("oracle_cg_f64", "oracle_cg_f32"):
                f = getattr(lib, name)
                f.restype = ctypes.c_int
                f.argtypes = [ctypes.c_int64, i64p, i32p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                              i64p, ctypes.c_int]
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _prep(u0: np.ndarray, offsets, weights, ndim):
    if u0.dtype not in (np.float32, np.float64):
        raise TypeError("oracle supports float32/float64 only")
    u0 = np.ascontiguousarray(u0)
    if ndim is None:
        ndim = u0.ndim
    shape = u0.shape
    if ndim == 2:
        if u0.ndim != 2:
            raise ValueError("2D oracle expects a [ny][nx] array")
        ext = (shape[1], shape[0], 1)
    elif ndim == 3:
        if u0.ndim != 3:
            raise ValueError("3D oracle expects a [nz][ny][nx] array")
        ext = (shape[2], shape[1], shape[0])
    else:
        raise ValueError("ndim must be 2 or 3")
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 3))
    # R6: weights rounded ONCE to the storage dtype (numpy casts round-to-nearest-even).
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).astype(u0.dtype))
    if w.shape[0] != offs.shape[0]:
        raise ValueError("offsets/weights length mismatch")
    return u0, ndim, np.asarray(ext, dtype=np.int64), offs, w


def run(u0: np.ndarray, offsets, weights, steps: int, bc: int = BC_FRAME,
        nthreads: int = 1, ndim: int | None = None) -> np.ndarray:
    """Return x^steps for initial field ``u0`` (C order [z][y][x] or [y][x])."""
    lib = _load()
    u0, ndim, ext, offs, w = _prep(u0, offsets, weights, ndim)
    out = np.empty_like(u0)
    fn = lib.oracle_stencil_f64 if u0.dtype == np.float64 else lib.oracle_stencil_f32
    st = fn(ndim, ext.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), offs.shape[0],
            offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), w.ctypes.data,
            int(bc), int(steps), u0.ctypes.data, out.ctypes.data, int(nthreads))
    if st != 0:
        raise OracleError(st)
    return out


def max_threads() -> int:
    return int(_load().oracle_max_threads())


# ---------------------------------------------------------------- CG (NEXT-3)
# cg_oracle.c: CSR SpMV and the conjugate-gradient Algorithm,
# readings RC1-RC4 in DESIGN.md.  Pins: tests/test_cg_oracle_pins.py.

def _csr(row_off, col, val, dtype):
    ro = np.ascontiguousarray(np.asarray(row_off, dtype=np.int64))
    ci = np.ascontiguousarray(np.asarray(col, dtype=np.int32))
    va = np.ascontiguousarray(np.asarray(val).astype(dtype, copy=False))
    n = ro.shape[0] - 1
    if n < 0 or ci.shape[0] != ro[-1] or va.shape[0] != ro[-1]:
        raise ValueError("inconsistent CSR arrays")
    return n, ro, ci, va


def csr_spmv(row_off, col, val, x: np.ndarray, nthreads: int = 1) -> np.ndarray:
    """y = A x, per row left to right with one fma per term in x's dtype."""
    lib = _load()
    x = np.ascontiguousarray(x)
    if x.dtype not in (np.float32, np.float64):
        raise TypeError("oracle supports float32/float64 only")
    n, ro, ci, va = _csr(row_off, col, val, x.dtype)
    if x.shape != (n,):
        raise ValueError("x has the wrong length")
    y = np.empty_like(x)
    fn = lib.oracle_csr_spmv_f64 if x.dtype == np.float64 else lib.oracle_csr_spmv_f32
    st = fn(n, ro.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), va.ctypes.data,
            x.ctypes.data, y.ctypes.data, int(nthreads))
    if st != 0:
        raise OracleError(st)
    return y


def cg(row_off, col, val, b: np.ndarray, kmax: int, tol: float = 0.0, nthreads: int = 1,
       allow_not_spd: bool = False):
    """Conjugate gradient from x0 = 0 (Algorithm, readings RC2-RC4).

    Returns ``(x, rr_history, iterations)`` with ``rr_history[k] = <r_k, r_k>`` for
    ``k = 0..iterations``.  A breakdown (<p,Ap> <= 0) raises OracleError(NOT_SPD)
    unless ``allow_not_spd`` (then the state at the breakdown is returned)."""
    lib = _load()
    b = np.ascontiguousarray(b)
    if b.dtype not in (np.float32, np.float64):
        raise TypeError("oracle supports float32/float64 only")
    n, ro, ci, va = _csr(row_off, col, val, b.dtype)
    if b.shape != (n,):
        raise ValueError("b has the wrong length")
    x = np.empty_like(b)
    hist = np.full(int(kmax) + 1, np.nan)
    it = np.zeros(1, dtype=np.int64)
    fn = lib.oracle_cg_f64 if b.dtype == np.float64 else lib.oracle_cg_f32
    st = fn(n, ro.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), va.ctypes.data, b.ctypes.data,
            int(kmax), float(tol), x.ctypes.data, hist.ctypes.data,
            it.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(nthreads))
    if st != 0 and not (st == 4 and allow_not_spd):
        raise OracleError(st)
    k = int(it[0])
    return x, hist[:k + 1], k
