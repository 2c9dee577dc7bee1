"""Run one stencil case on the GPU and compare with the oracle (dev aid).
    python tools/dbg_case.py 3d7pt 34,40,132 f32 hostloop 1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil

name, shape, dt, variant, T = sys.argv[1], tuple(int(v) for v in sys.argv[2].split(",")), sys.argv[3], sys.argv[4], int(sys.argv[5])
dtype = np.float32 if dt == "f32" else np.float64
offs, w = si.preset(name)
u0 = si.field(shape, dtype=dtype, seed=202)
st = Stencil(shape, offs, w, dtype=dtype)
print(st.query(variant))
x = torch.from_numpy(u0).cuda()
out = st.run(x, T, variant)
torch.cuda.synchronize()
ref = oracle.run(u0, offs, w, T)
got = out.cpu().numpy()
bad = np.argwhere(got != ref)
print("mismatches:", len(bad), bad[:10])
