"""Multi-GPU paths on real devices; skipped when fewer than 2 GPUs are visible
(the single-GPU emulation of the slab exchange is tests/test_gpu_dist.py, the host-side logic
tests/test_dist_host.py).

* cross-device, same process: two slab handles on cuda:0 and cuda:1 connected with
  perks_stencil_dist_connect (peer pointers, P2P stores over NVLink), persistent and PERKS kernels
  launched on both devices before either is synchronised; the gathered result must equal the CPU
  oracle on the global domain bit-exactly (reading R12);
* the NCCL host-loop baseline (paper_2204_02064_b200/nccl_slab.py) with the nccl backend and the
  CUDA library as the step, two processes, one GPU each.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _need_two():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")


@pytest.mark.parametrize("variant", ["hostloop", "persistent", "perks"])
@pytest.mark.parametrize("name,dtype", [("3d7pt", np.float64), ("3d27pt", np.float32)])
def test_two_devices_same_process_peer_exchange(variant, name, dtype):
    _need_two()
    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200.dist import slab_bounds

    shape, T = (40, 36, 64), 7
    offs, w = si.preset(name)
    u0 = si.field(shape, dtype=dtype)
    sts, xs, outs = [], [], []
    for r in range(2):
        z0, z1 = slab_bounds(shape[0], 2, r)
        st = Stencil((z1 - z0,) + shape[1:], offs, w, dtype=dtype, device=r, rank=r, nranks=2)
        sts.append(st)
        xs.append(torch.from_numpy(u0[z0:z1]).to(f"cuda:{r}"))
        outs.append(torch.full_like(xs[-1], float("nan")))
    blobs = [st.export_blob() for st in sts]
    sts[0].connect(None, blobs[1])
    sts[1].connect(blobs[0], None)
    for r in range(2):  # both launched before either is synchronised (they wait on each other)
        with torch.cuda.device(r):
            sts[r].run(xs[r], T, variant, out=outs[r])
    for r in range(2):
        torch.cuda.synchronize(r)
    got = np.concatenate([o.cpu().numpy() for o in outs])
    assert np.array_equal(got, oracle.run(u0, offs, w, T))
    for st in sts:
        st.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_worker(rank, world, port, q, name, shape, steps, dtype):
    import torch.distributed as dist

    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200.nccl_slab import NcclSlabHostLoop

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    offs, w = si.preset(name)
    radius = max(max(abs(v) for v in o) for o in offs)
    u0 = si.field(shape, dtype=dtype)
    holder = {}

    def empty(s):
        return torch.zeros(s, dtype=torch.float64 if dtype == np.float64 else torch.float32, device=f"cuda:{rank}")

    def step(src, dst):
        if "st" not in holder:
            holder["st"] = Stencil(tuple(src.shape), offs, w, dtype=dtype, device=rank)
        holder["st"].run(src, 1, "hostloop", out=dst)

    sl = NcclSlabHostLoop(shape, radius, rank, world, step, empty)
    sl.load(torch.from_numpy(u0[sl.z0:sl.z1]).to(f"cuda:{rank}"))
    out = sl.run(steps).cpu().numpy().copy()
    q.put((rank, sl.z0, sl.z1, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,dtype,shape", [("3d7pt", np.float64, (24, 20, 32)), ("3d27pt", np.float32, (24, 20, 32)),
                                              ("2d9pt", np.float32, (40, 64))])
def test_nccl_slab_hostloop_two_gpus(name, dtype, shape):
    _need_two()
    import torch.multiprocessing as mp

    world, steps = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, q, name, shape, steps, dtype)) for r in range(world)]
    for p in ps:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    offs, w = si.preset(name)
    ref = oracle.run(si.field(shape, dtype=dtype), offs, w, steps)
    got = np.empty_like(ref)
    for _, z0, z1, out in parts:
        got[z0:z1] = out
    assert np.array_equal(got, ref)
