"""One general-3D (k3d_wide.cu) run for ncu: prof_wide3.py VARIANT T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil
offs, w = si.preset("3d13pt")
st = Stencil((256, 256, 256), offs, w, dtype=np.float64)
x = si.field_torch((256, 256, 256), np.float64, "cuda")
st.run(x, int(sys.argv[2]), sys.argv[1])
torch.cuda.synchronize()
