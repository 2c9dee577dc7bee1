"""Python API over the C ABI: ``Stencil`` handle + ``run`` convenience.

PyTorch is used only for device memory and streams (tensors are passed to the library as raw
device pointers on ``torch.cuda.current_stream()``).  Every stencil step runs in
libperks_stencil.so; nothing here computes.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import VARIANTS, check, lib
from .dist import exchange_neighbour_blobs


def _dtype_code(dtype) -> int:
    import torch

    if dtype in ("f32", "float32", np.float32, torch.float32):
        return _lib.F32
    if dtype in ("f64", "float64", np.float64, torch.float64):
        return _lib.F64
    raise TypeError(f"unsupported dtype {dtype!r} (f32/f64 only)")


def _variant(v) -> int:
    if isinstance(v, int):
        return v
    return VARIANTS[v]


class Stencil:
    """Handle for one (domain, point set, dtype, bc) on one device.

    shape: C-order extents, (ny, nx) for 2D or (nz, ny, nx) for 3D.
    offsets: list of (dx, dy, dz); list order = accumulation order (reading R5).
    weights: floats, rounded once to dtype by the library (reading R6).
    """

    def __init__(self, shape, offsets, weights, dtype="f64", bc="frame", device=0, rank=0,
                 nranks=1):
        """rank/nranks > 1: this handle is rank's z-slab of a slab-decomposed global domain
        (perks_stencil_create_dist); ``shape`` is the LOCAL slab.  Connect it with
        ``connect`` (or ``connect_torch_distributed``) before running."""
        shape = tuple(int(s) for s in shape)
        if len(shape) not in (2, 3):
            raise ValueError("shape must be (ny, nx) or (nz, ny, nx)")
        self.shape = shape
        self.ndim = len(shape)
        ext = (shape[-1], shape[-2], shape[0] if self.ndim == 3 else 1)
        offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 3))
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
        self._offs, self._w = offs, w  # keep alive during create
        d = _lib.Desc()
        d.ndim = self.ndim
        d.extent[:] = ext
        d.npoints = offs.shape[0]
        d.offsets = offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        d.weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.dtype = _dtype_code(dtype)
        d.bc = {"frame": _lib.BC_FRAME, "periodic": _lib.BC_PERIODIC}[bc] if isinstance(bc, str) else int(bc)
        self.dtype_code = d.dtype
        self.device = int(device)
        h = ctypes.c_void_p()
        self.rank, self.nranks = int(rank), int(nranks)
        if self.nranks > 1:
            check(lib.perks_stencil_create_dist(ctypes.byref(d), self.device, self.rank,
                                                self.nranks, ctypes.byref(h)),
                  "perks_stencil_create_dist")
        else:
            check(lib.perks_stencil_create(ctypes.byref(d), self.device, ctypes.byref(h)),
                  "perks_stencil_create")
        self._h = h
        self._ws = {}

    # ------------------------------------------------------------------ info
    @property
    def torch_dtype(self):
        import torch

        return torch.float64 if self.dtype_code == _lib.F64 else torch.float32

    @property
    def np_dtype(self):
        return np.float64 if self.dtype_code == _lib.F64 else np.float32

    def workspace_bytes(self, variant="auto") -> int:
        b = ctypes.c_size_t()
        check(lib.perks_stencil_workspace_bytes(self._h, _variant(variant), ctypes.byref(b)),
              "perks_stencil_workspace_bytes")
        return int(b.value)

    def query(self, variant="auto") -> dict:
        info = _lib.PlanInfo()
        check(lib.perks_stencil_query(self._h, _variant(variant), ctypes.byref(info)),
              "perks_stencil_query")
        return {
            "variant": _lib.VARIANT_NAMES[info.variant], "grid": info.grid, "block": info.block,
            "ctas_per_sm": info.ctas_per_sm, "tile": list(info.tile),
            "regs_per_thread": info.regs_per_thread, "smem_per_cta": info.smem_per_cta,
            "cached_cells_reg": info.cached_cells_reg, "cached_cells_smem": info.cached_cells_smem,
            "cached_cells_tmem": info.cached_cells_tmem, "tmem_cols_per_cta": info.tmem_cols_per_cta,
            "total_cells": info.total_cells, "dram_bytes_per_step": info.dram_bytes_per_step,
            "halo_bytes_per_step": info.halo_bytes_per_step,
            "workspace_bytes": int(info.workspace_bytes),
            "kernel": info.kernel_name.decode(),
        }

    def launch_count(self, variant, steps) -> int:
        n = ctypes.c_int64()
        check(lib.perks_stencil_launch_count(self._h, _variant(variant), int(steps), ctypes.byref(n)),
              "perks_stencil_launch_count")
        return int(n.value)

    # ------------------------------------------------------------------ run
    def workspace(self, variant="auto"):
        """Cached device workspace (torch uint8 tensor, 256-B aligned by the caching allocator)."""
        import torch

        v = _variant(variant)
        nb = self.workspace_bytes(v)
        ws = self._ws.get(v)
        if ws is None or ws.numel() < nb:
            ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws[v] = ws
        return ws

    def run(self, x, steps: int, variant="auto", out=None, workspace=None, stream=None):
        """Enqueue ``steps`` steps on the current torch stream; returns ``out``."""
        import torch

        self._check_device_tensor(x, "x")
        if out is None:
            out = torch.empty_like(x)
        else:
            self._check_device_tensor(out, "out")
        v = _variant(variant)
        ws = workspace
        if ws is None and steps > 0:
            ws = self.workspace(v)
        s = stream if stream is not None else torch.cuda.current_stream(x.device)
        check(lib.perks_stencil_run(
            self._h, v, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(ws.data_ptr() if ws is not None else 0),
            ctypes.c_size_t(ws.numel() if ws is not None else 0), int(steps),
            ctypes.c_void_p(s.cuda_stream)), "perks_stencil_run")
        return out

    def _check_device_tensor(self, t, what):
        """A CUDA tensor of the handle's shape and dtype, dense, on the handle's device (the
        library reads/writes cells*elem bytes through its pointer)."""
        import torch

        if not (isinstance(t, torch.Tensor) and t.is_cuda):
            raise TypeError(f"{what} must be a CUDA tensor (use run_host for host arrays)")
        if tuple(t.shape) != self.shape or t.dtype != self.torch_dtype or not t.is_contiguous():
            raise ValueError(f"{what} must be a contiguous tensor of the handle's shape {self.shape} "
                             f"and dtype {self.torch_dtype}")
        if (t.device.index or 0) != self.device:
            raise ValueError(f"{what} is on cuda:{t.device.index}, the handle on cuda:{self.device}")

    def _check_host_array(self, a, what):
        """A C-contiguous CPU array/tensor of the handle's shape and dtype (run_host copies
        cells*elem bytes through its raw pointer)."""
        import torch

        if isinstance(a, np.ndarray):
            ok = (a.shape == self.shape and a.dtype == self.np_dtype and a.flags.c_contiguous)
        elif isinstance(a, torch.Tensor):
            if a.is_cuda:
                raise TypeError(f"{what} must be host memory (use run() for CUDA tensors)")
            ok = (tuple(a.shape) == self.shape and a.dtype == self.torch_dtype and a.is_contiguous())
        else:
            raise TypeError(f"{what} must be a numpy array or a CPU torch tensor")
        if not ok:
            raise ValueError(f"{what} must be C-contiguous with the handle's shape {self.shape} and "
                             f"dtype {np.dtype(self.np_dtype).name}")

    def run_host(self, x_host, steps: int, variant="auto", out=None):
        """End-to-end call with host buffers (H2D, run, D2H, synchronise) — blocking."""
        import torch

        self._check_host_array(x_host, "x_host")
        if out is not None:
            self._check_host_array(out, "out")
        if isinstance(x_host, np.ndarray):
            src = x_host
            dst = np.empty_like(src) if out is None else out
            p_in, p_out = src.ctypes.data, dst.ctypes.data
        else:
            src = x_host
            dst = torch.empty_like(src) if out is None else out
            p_in, p_out = src.data_ptr(), dst.data_ptr()
        check(lib.perks_stencil_run_host(self._h, _variant(variant), ctypes.c_void_p(p_in),
                                         ctypes.c_void_p(p_out), int(steps)),
              "perks_stencil_run_host")
        return dst

    # ------------------------------------------------------------------ multi-GPU slabs
    def export_blob(self) -> bytes:
        """This rank's connection blob (IPC handle of the library-owned ghost planes)."""
        buf = ctypes.create_string_buffer(_lib.DIST_BLOB_BYTES)
        check(lib.perks_stencil_dist_export(self._h, buf), "perks_stencil_dist_export")
        return buf.raw

    def connect(self, lower_blob, upper_blob):
        """Connect to rank-1 / rank+1 (None where there is no neighbour)."""
        lo = ctypes.create_string_buffer(lower_blob, len(lower_blob)) if lower_blob else None
        hi = ctypes.create_string_buffer(upper_blob, len(upper_blob)) if upper_blob else None
        check(lib.perks_stencil_dist_connect(self._h, lo, hi), "perks_stencil_dist_connect")

    def connect_torch_distributed(self, group=None):
        """Exchange blobs with torch.distributed (plumbing only) and connect."""
        lower, upper = exchange_neighbour_blobs(self.export_blob(), group)
        self.connect(lower, upper)

    def close(self):
        if getattr(self, "_h", None):
            lib.perks_stencil_destroy(self._h)
            self._h = None
        self._ws = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(x, offsets, weights, steps, variant="auto", bc="frame"):
    """One-shot: build a handle for ``x``'s shape/dtype and return x^steps (new tensor)."""
    st = Stencil(tuple(x.shape), offsets, weights, dtype=x.dtype, bc=bc,
                 device=x.device.index or 0)
    try:
        return st.run(x, steps, variant)
    finally:
        import torch

        torch.cuda.current_stream(x.device).synchronize()
        st.close()


def run_group(stencils, xs, steps, variant="auto", outs=None, stream=None):
    """Run the connected slab handles ``stencils`` (all on ONE device) together — the single-GPU
    emulation of a multi-GPU slab decomposition (perks_stencil_run_group)."""
    import torch

    n = len(stencils)
    if len(xs) != n or (outs is not None and len(outs) != n):
        raise ValueError("run_group: one input (and output) per handle")
    for st, x in zip(stencils, xs):
        st._check_device_tensor(x, "xs[i]")
    if outs is None:
        outs = [torch.empty_like(x) for x in xs]
    else:
        for st, o in zip(stencils, outs):
            st._check_device_tensor(o, "outs[i]")
    v = _variant(variant)
    wss = [st.workspace(v) for st in stencils]
    VP = ctypes.c_void_p
    hs = (VP * n)(*[st._h for st in stencils])
    ins = (VP * n)(*[x.data_ptr() for x in xs])
    os_ = (VP * n)(*[o.data_ptr() for o in outs])
    ws = (VP * n)(*[w.data_ptr() for w in wss])
    wb = (ctypes.c_size_t * n)(*[w.numel() for w in wss])
    s = stream if stream is not None else torch.cuda.current_stream(xs[0].device)
    check(lib.perks_stencil_run_group(hs, n, v, ins, os_, ws, wb, int(steps), VP(s.cuda_stream)),
          "perks_stencil_run_group")
    return outs
