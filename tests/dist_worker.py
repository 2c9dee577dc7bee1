"""Single-GPU emulation of the multi-GPU slab decomposition (run in a child process by
tests/test_gpu_dist.py so that a watchdog trap cannot poison the test process).

usage: python dist_worker.py OUT.npy NAME NZ NY NX DTYPE NRANKS VARIANT[,VARIANT...] T1 [T2 ...]
Splits the seeded global field into NRANKS z-slabs (one Stencil handle each, all on cuda:0),
connects the chain, runs T1, then T2, ... steps back to back (each run feeds the next), and saves
the concatenated global result."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402


def main(argv):
    out_path, name = argv[0], argv[1]
    nz, ny, nx = (int(a) for a in argv[2:5])
    dtype = np.float64 if argv[5] == "f64" else np.float32
    n, variant = int(argv[6]), argv[7]
    Ts = [int(a) for a in argv[8:]]
    os.environ.setdefault("PERKS_NUM_SMS", str(max(1, 148 // n)))  # all slabs resident together
    import torch

    import seeded_inputs as si
    from paper_2204_02064_b200 import Stencil, run_group
    from paper_2204_02064_b200.dist import slab_bounds

    offs, w = si.preset(name)
    u0 = si.field((nz, ny, nx), dtype=dtype, seed=505)
    sts, xs = [], []
    for r in range(n):
        z0, z1 = slab_bounds(nz, n, r)
        sts.append(Stencil((z1 - z0, ny, nx), offs, w, dtype=dtype, rank=r, nranks=n))
        xs.append(torch.from_numpy(np.ascontiguousarray(u0[z0:z1])).cuda())
    blobs = [st.export_blob() for st in sts]
    for r, st in enumerate(sts):
        st.connect(blobs[r - 1] if r > 0 else None, blobs[r + 1] if r < n - 1 else None)
    variants = variant.split(",")  # one variant for every run, or one per run (mixed on the same handles)
    for i, T in enumerate(Ts):
        outs = [torch.full_like(x, float("nan")) for x in xs]
        run_group(sts, xs, T, variants[i % len(variants)], outs=outs)
        torch.cuda.synchronize()
        xs = outs
    res = np.concatenate([x.cpu().numpy() for x in xs], axis=0)
    np.save(out_path, res)
    for st in sts:
        st.close()


if __name__ == "__main__":
    main(sys.argv[1:])
