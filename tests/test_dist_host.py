"""Host-side logic of the multi-GPU slab decomposition, on CPU: slab bounds and the one-time
neighbour blob exchange over torch.distributed (gloo, world_size 2 and 3, 127.0.0.1)."""
import os
import socket

import pytest

from paper_2204_02064_b200.dist import exchange_neighbour_blobs, slab_bounds


def test_slab_bounds_cover_domain():
    for nz in (2, 7, 1024, 3000):
        for n in (1, 2, 3, 8):
            if nz < n:
                continue
            b = [slab_bounds(nz, n, r) for r in range(n)]
            assert b[0][0] == 0 and b[-1][1] == nz
            assert all(b[r][1] == b[r + 1][0] for r in range(n - 1))
            sizes = [z1 - z0 for z0, z1 in b]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank]) * 128
    lo, hi = exchange_neighbour_blobs(blob)
    q.put((rank, lo, hi))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_blob_exchange_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, lo, hi = q.get(timeout=120)
        res[r] = (lo, hi)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        lo, hi = res[r]
        assert lo == (bytes([r - 1]) * 128 if r > 0 else None)
        assert hi == (bytes([r + 1]) * 128 if r < world - 1 else None)


# ---------------------------------------------------------------- NCCL host-loop slab baseline
# per-step halo send/recv + one host-loop step per time step.  The exchange logic
# runs here on CPU with gloo and the CPU oracle as the step; the gathered slabs must equal the
# oracle on the global domain bit-exactly (reading R12) — on GPU the same class drives NCCL and
# the CUDA library (bench.py --variant nccl).

def _nccl_slab_worker(rank, world, port, q, name, shape, steps):
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import seeded_inputs as si
    from paper_2204_02064_b200.nccl_slab import NcclSlabHostLoop

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    offs, w = si.preset(name)
    r = max(max(abs(v) for v in o) for o in offs)
    u0 = si.field(shape, dtype=np.float64)

    def step(src, dst):
        dst.copy_(torch.from_numpy(oracle.run(src.numpy(), offs, w, 1)))

    sl = NcclSlabHostLoop(shape, r, rank, world, step, lambda s: torch.zeros(s, dtype=torch.float64))
    sl.load(torch.from_numpy(u0[sl.z0:sl.z1]))
    out = sl.run(steps).numpy().copy()
    q.put((rank, sl.z0, sl.z1, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name,shape,steps", [(2, "3d7pt", (9, 6, 7), 5), (3, "3d27pt", (11, 5, 6), 4),
                                                     (2, "3d13pt", (12, 7, 7), 3),
                                                     # 2D: y-slabs, radius 1 and 3
                                                     (2, "2d9pt", (13, 10), 6), (3, "2d5pt", (14, 9), 5),
                                                     (2, "2d13pt", (17, 12), 4)])
def test_nccl_slab_hostloop_matches_global_oracle(world, name, shape, steps):
    import numpy as np
    import torch.multiprocessing as mp

    import oracle
    import seeded_inputs as si

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_slab_worker, args=(r, world, port, q, name, shape, steps)) for r in range(world)]
    for p in ps:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    offs, w = si.preset(name)
    ref = oracle.run(si.field(shape, dtype=np.float64), offs, w, steps)
    got = np.empty_like(ref)
    for _, z0, z1, out in parts:
        got[z0:z1] = out
    assert np.array_equal(got, ref)
