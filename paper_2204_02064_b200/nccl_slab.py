"""The multi-GPU host-loop baseline of SURVEY §8(e)(a): slabs along the slowest axis (z in 3D, y in
2D, SURVEY §8(b) "global z split evenly; y for 2D"), halo planes / rows exchanged every step by NCCL
send/recv (torch.distributed point-to-point on the "nccl" backend), one host-loop stencil step per
time step through the C ABI.

This is the baseline the in-kernel exchange of the persistent / PERKS slab path (csrc/dist.cuh,
``Stencil(..., rank, nranks)``) is measured against.  Layout: rank r owns global planes
[z0, z1) (``dist.slab_bounds``) and keeps them in an *extended* slab with ``h = r_stencil`` halo
planes below (if r > 0) and above (if r < N-1).  A step is

    1. send my first h owned planes down and my last h owned planes up, receive the neighbours'
       planes into my halo planes (one batch of isend/irecv, ncclGroupStart/End underneath);
    2. one stencil step on the extended slab (``perks_stencil_run``, host-loop variant, T = 1):
       the FRAME boundary (reading R1) keeps the extended slab's outer planes fixed — the halo
       planes of an interior face, the global frame planes of rank 0 / rank N-1 — so the owned
       planes are updated exactly as in the single-GPU run on the global domain (reading R12).

The class is written against two callables (a step function and the torch.distributed group), so
the exchange logic is tested on CPU with the gloo backend and the CPU oracle as the step
(tests/test_dist_host.py); on a GPU the step is the CUDA library.  Nothing here computes stencil
arithmetic.
"""
from __future__ import annotations

from .dist import slab_bounds


class NcclSlabHostLoop:
    """One rank of a slab decomposition along axis 0 (z of [nz][ny][nx], y of [ny][nx]) with
    per-step halo send/recv.

    global_shape: (nz, ny, nx) or (ny, nx).  step(src, dst): advance the extended slab ``src`` by
    one time step into ``dst`` (same shape); on GPU a ``Stencil(...).run(src, 1, "hostloop",
    out=dst)``.  z0/z1/nz name the slab's range along axis 0 in either case.
    """

    def __init__(self, global_shape, radius: int, rank: int, nranks: int, step, empty, group=None):
        global_shape = tuple(int(v) for v in global_shape)
        if len(global_shape) not in (2, 3):
            raise ValueError("global_shape must be (nz, ny, nx) or (ny, nx)")
        self.rank, self.nranks, self.h = int(rank), int(nranks), int(radius)
        self.z0, self.z1 = slab_bounds(global_shape[0], nranks, rank)
        self.nz = self.z1 - self.z0
        if self.nz < self.h:
            raise ValueError("slab thinner than the stencil radius")
        self.lo = self.h if rank > 0 else 0
        self.hi = self.h if rank < nranks - 1 else 0
        self.shape = (self.lo + self.nz + self.hi,) + global_shape[1:]
        self.step = step
        self.group = group
        self.a = empty(self.shape)
        self.b = empty(self.shape)

    def owned(self, buf=None):
        """The owned planes of an extended buffer (a view)."""
        buf = self.a if buf is None else buf
        return buf[self.lo:self.lo + self.nz]

    def load(self, local):
        """Set the owned planes (the rank's [z0, z1) part of the global field)."""
        self.owned(self.a).copy_(local)

    def exchange(self, buf):
        """Halo planes of ``buf`` from the neighbours: one batch of point-to-point sends and
        receives (ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd on the nccl backend).
        Slices along axis 0 of a C-order slab are contiguous, so planes (rows in 2D) go straight from
        / into the extended buffer."""
        import torch.distributed as dist

        ops = []
        h, lo, nz = self.h, self.lo, self.nz
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, buf[lo:lo + h], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[0:h], self.rank - 1, self.group))
        if self.rank < self.nranks - 1:
            ops.append(dist.P2POp(dist.isend, buf[lo + nz - h:lo + nz], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, buf[lo + nz:lo + nz + h], self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def run(self, steps: int):
        """Advance the owned planes ``steps`` time steps; returns the owned planes (a view)."""
        for _ in range(int(steps)):
            self.exchange(self.a)
            self.step(self.a, self.b)
            self.a, self.b = self.b, self.a
        return self.owned(self.a)
