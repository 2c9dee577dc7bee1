"""Host-side plumbing of the multi-GPU slab decomposition.

Only connection set-up lives here: each rank's library exports a small blob (an IPC handle of its
ghost planes), and torch.distributed carries the blobs to the neighbours once.  The per-step halo
exchange itself runs inside the CUDA kernels (csrc/dist.cuh) — no collective is on the data path.
This module does not load the CUDA library, so it is testable on CPU with the gloo backend.
"""
from __future__ import annotations


def exchange_neighbour_blobs(blob: bytes, group=None):
    """all_gather every rank's blob over torch.distributed; return (lower, upper) neighbour blobs
    of the calling rank along the slab chain (None at the chain ends)."""
    import torch.distributed as dist

    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    blobs = [None] * ws
    dist.all_gather_object(blobs, bytes(blob), group=group)
    lower = blobs[rank - 1] if rank > 0 else None
    upper = blobs[rank + 1] if rank < ws - 1 else None
    return lower, upper



def slab_bounds(nz_global: int, nranks: int, rank: int):
    """[z0, z1) of rank's slab when nz_global planes are split as evenly as possible along z."""
    base, extra = divmod(int(nz_global), int(nranks))
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)
