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
