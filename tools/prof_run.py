"""Run one config/variant a few times (for ncu capture). Usage: prof_run.py C2 perks [T] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil
cn, v = sys.argv[1], sys.argv[2]
c = si.CONFIGS[cn]
T = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else c["steps"]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
dt = np.float64 if c["dtype"] == "f64" else np.float32
offs, w = si.preset(c["stencil"])
st = Stencil(c["shape"], offs, w, dtype=dt)
x = si.field_torch(c["shape"], dt, "cuda")
out = torch.empty_like(x)
for _ in range(reps):
    st.run(x, T, v, out=out)
torch.cuda.synchronize()
print(st.query(v))
