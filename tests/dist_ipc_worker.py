"""One rank of a 2-process slab decomposition on ONE GPU (tests/test_gpu_dist.py): the ranks are
separate processes, so each maps its neighbour's ghost planes through cudaIpcOpenMemHandle (the
cross-process path a multi-GPU run takes), with the blobs carried by torch.distributed (gloo).

usage: python dist_ipc_worker.py OUT_PREFIX NAME NZ NY NX DTYPE VARIANT T1 [T2 ...]
(RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT from the environment)"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402


def main(argv):
    prefix, name = argv[0], argv[1]
    nz, ny, nx = (int(a) for a in argv[2:5])
    dtype = np.float64 if argv[5] == "f64" else np.float32
    variant = argv[6]
    Ts = [int(a) for a in argv[7:]]
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    import torch
    import torch.distributed as dist

    import seeded_inputs as si
    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200.dist import slab_bounds

    dist.init_process_group("gloo", rank=rank, world_size=n)
    offs, w = si.preset(name)
    z0, z1 = slab_bounds(nz, n, rank)
    u0 = si.field((nz, ny, nx), dtype=dtype, seed=505)
    st = Stencil((z1 - z0, ny, nx), offs, w, dtype=dtype, rank=rank, nranks=n, device=0)
    st.connect_torch_distributed()
    x = torch.from_numpy(np.ascontiguousarray(u0[z0:z1])).cuda()
    for T in Ts:
        out = torch.full_like(x, float("nan"))
        st.run(x, T, variant, out=out)
        torch.cuda.synchronize()
        x = out
    np.save(f"{prefix}{rank}.npy", x.cpu().numpy())
    dist.barrier()
    st.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1:])
