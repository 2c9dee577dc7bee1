"""Emulated slab timing on ONE GPU (dev aid): N slab handles of a global 3D 7-point domain run together
through run_group (each slab on its own stream, SMs split by PERKS_NUM_SMS).  Not a multi-GPU number:
the slabs share one GPU's HBM and SMs.  usage: dist_timing.py NZ NY NX f64|f32 N T variant"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
nz, ny, nx = (int(a) for a in sys.argv[1:4])
n, T, variant = int(sys.argv[5]), int(sys.argv[6]), sys.argv[7]
os.environ.setdefault("PERKS_NUM_SMS", str(max(1, 148 // n)))
import numpy as np, torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil, run_group
from paper_2204_02064_b200.dist import slab_bounds
dt = np.float64 if sys.argv[4] == "f64" else np.float32
offs, w = si.preset("3d7pt")
sts, xs = [], []
for r in range(n):
    z0, z1 = slab_bounds(nz, n, r)
    sts.append(Stencil((z1 - z0, ny, nx), offs, w, dtype=dt, rank=r, nranks=n))
    xs.append(si.field_torch((z1 - z0, ny, nx), dt, "cuda"))
blobs = [st.export_blob() for st in sts]
for r, st in enumerate(sts):
    st.connect(blobs[r - 1] if r > 0 else None, blobs[r + 1] if r < n - 1 else None)
outs = [torch.empty_like(x) for x in xs]
run_group(sts, xs, 2, variant, outs=outs)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run_group(sts, xs, T, variant, outs=outs); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / T)
print(f"{n} slabs of {nz}x{ny}x{nx} {sys.argv[4]} {variant} kernel={sts[0].query(variant)['kernel']} "
      f"PERKS_TB_DIST={os.environ.get('PERKS_TB_DIST', '1')}: best {min(ts):.2f} median {statistics.median(ts):.2f} us/step")
