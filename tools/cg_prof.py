"""One CG solve for ncu: python tools/cg_prof.py WL VARIANT POLICY K"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import seeded_inputs.sparse as sp  # noqa: E402
from paper_2204_02064_b200 import CG  # noqa: E402

wl, v, p, K = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
kind, size, dtype, _, _ = sp.CG_WORKLOADS[wl]
ro, ci, va = sp.matrix(kind, size)
h = CG(ro, ci, va, dtype="f64" if dtype == np.float64 else "f32")
b = torch.from_numpy(sp.rhs(len(ro) - 1, dtype=dtype)).cuda()
x, hist, info = h.solve(b, K, 0.0, v, p)
torch.cuda.synchronize()
print(wl, v, p, "iters", int(info[0]))
