"""Python API over the CG C ABI (include/perks/perks_cg.h): the ``CG`` handle.

Argument marshalling only: the SpMV, the inner products, the vector updates and the iteration
loop run in libperks_stencil.so (csrc/cg.cu).  PyTorch provides device memory and streams.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import CG_POLICIES, VARIANTS, check, lib


def _policy(p) -> int:
    return p if isinstance(p, int) else CG_POLICIES[p]


def _variant(v) -> int:
    return v if isinstance(v, int) else VARIANTS[v]


class CG:
    """A CSR matrix on one device, ready for CG solves (Algorithm).

    row_off: n+1 int64 offsets; col: nnz int32 columns; val: nnz values (rounded once to
    ``dtype`` by the library)."""

    def __init__(self, row_off, col, val, dtype="f64", device=0):
        ro = np.ascontiguousarray(np.asarray(row_off, dtype=np.int64))
        ci = np.ascontiguousarray(np.asarray(col, dtype=np.int32))
        va = np.ascontiguousarray(np.asarray(val, dtype=np.float64))
        n = ro.shape[0] - 1
        if n < 0 or ci.shape[0] != va.shape[0]:
            raise ValueError("inconsistent CSR arrays")
        self.n, self.nnz = int(n), int(ci.shape[0])
        self.dtype_code = {"f32": _lib.F32, "float32": _lib.F32, np.float32: _lib.F32,
                           "f64": _lib.F64, "float64": _lib.F64, np.float64: _lib.F64}[dtype]
        self.np_dtype = np.float64 if self.dtype_code == _lib.F64 else np.float32
        self.device = int(device)
        d = _lib.CsrDesc()
        d.n_rows = self.n
        d.nnz = self.nnz
        d.row_offsets = ro.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        d.col_indices = ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.values = va.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.dtype = self.dtype_code
        h = ctypes.c_void_p()
        check(lib.perks_cg_create(ctypes.byref(d), self.device, ctypes.byref(h)), "perks_cg_create")
        self._h = h
        self._ws = None

    @property
    def torch_dtype(self):
        import torch

        return torch.float64 if self.dtype_code == _lib.F64 else torch.float32

    def workspace(self):
        import torch

        if self._ws is None:
            nb = ctypes.c_size_t()
            check(lib.perks_cg_workspace_bytes(self._h, ctypes.byref(nb)), "perks_cg_workspace_bytes")
            self._ws = torch.empty(max(int(nb.value), 256), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def _check_vec(self, t, name):
        import torch

        if not isinstance(t, torch.Tensor) or t.dtype != self.torch_dtype or t.shape != (self.n,) \
                or not t.is_contiguous() or t.device != torch.device(f"cuda:{self.device}"):
            raise ValueError(f"{name} must be a contiguous {self.torch_dtype} tensor of shape ({self.n},) "
                             f"on cuda:{self.device}")

    def spmv(self, x, out=None):
        """y = A x (merge-based SpMV kernel, one launch) on the current stream."""
        import torch

        self._check_vec(x, "x")
        y = torch.empty_like(x) if out is None else out
        self._check_vec(y, "out")
        ws = self.workspace()
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(lib.perks_cg_spmv(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(s)),
              "perks_cg_spmv")
        return y

    def solve(self, b, kmax: int, tol: float = 0.0, variant="perks", policy="auto", out=None,
              history=None, info=None):
        """Enqueue a CG solve from x0 = 0 on the current stream.  Returns (x, history, info)
        device tensors: history[k] = <r_k, r_k> (float64, kmax+1), info = [iterations, status]."""
        import torch

        self._check_vec(b, "b")
        x = torch.empty_like(b) if out is None else out
        self._check_vec(x, "out")
        dev = f"cuda:{self.device}"
        if history is None:
            history = torch.full((int(kmax) + 1,), float("nan"), dtype=torch.float64, device=dev)
        if info is None:
            info = torch.zeros(2, dtype=torch.int64, device=dev)
        if (history.numel() < kmax + 1 or history.dtype != torch.float64 or not history.is_contiguous()
                or history.device != torch.device(dev)):
            raise ValueError(f"history must be a contiguous float64 tensor of >= kmax+1 values on {dev}")
        if info.numel() < 2 or info.dtype != torch.int64 or not info.is_contiguous() or info.device != torch.device(dev):
            raise ValueError(f"info must be a contiguous int64 tensor of >= 2 values on {dev}")
        ws = self.workspace()
        s = torch.cuda.current_stream(self.device).cuda_stream
        check(lib.perks_cg_solve(self._h, _variant(variant), _policy(policy), ctypes.c_void_p(b.data_ptr()),
                                 ctypes.c_void_p(x.data_ptr()), int(kmax), float(tol),
                                 ctypes.c_void_p(history.data_ptr()), ctypes.c_void_p(info.data_ptr()),
                                 ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(s)),
              "perks_cg_solve")
        return x, history, info

    def solve_host(self, b: np.ndarray, kmax: int, tol: float = 0.0, variant="perks", policy="auto"):
        """End to end through perks_cg_solve_host: host b in, host (x, history, iterations, status)."""
        b = np.ascontiguousarray(b)
        if b.dtype != self.np_dtype or b.shape != (self.n,):
            raise ValueError(f"b must be a C-contiguous {self.np_dtype.__name__} array of shape ({self.n},)")
        x = np.empty_like(b)
        hist = np.full(int(kmax) + 1, np.nan)
        info = np.zeros(2, dtype=np.int64)
        check(lib.perks_cg_solve_host(self._h, _variant(variant), _policy(policy), ctypes.c_void_p(b.ctypes.data),
                                      ctypes.c_void_p(x.ctypes.data), int(kmax), float(tol),
                                      ctypes.c_void_p(hist.ctypes.data), ctypes.c_void_p(info.ctypes.data)),
              "perks_cg_solve_host")
        return x, hist, int(info[0]), int(info[1])

    def query(self, variant="perks", policy="auto") -> dict:
        inf = _lib.CgInfo()
        check(lib.perks_cg_query(self._h, _variant(variant), _policy(policy), ctypes.byref(inf)), "perks_cg_query")
        out = {f: getattr(inf, f) for f, _ in _lib.CgInfo._fields_}
        out["kernel_name"] = inf.kernel_name.decode()
        out["variant"] = _lib.VARIANT_NAMES[inf.variant]
        out["policy"] = _lib.CG_POLICY_NAMES[inf.policy]
        return out

    def partition(self) -> np.ndarray:
        g = self.query("persistent", "imp")["grid"]
        rows = np.zeros(g + 1, dtype=np.int64)
        check(lib.perks_cg_partition(self._h, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), g + 1),
              "perks_cg_partition")
        return rows

    def close(self):
        if getattr(self, "_h", None):
            lib.perks_cg_destroy(self._h)
            self._h = None
        self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
