"""Time one shape/stencil/variant (dev aid): python tools/run_shape.py NZ,NY,NX f64 3d7pt T v1,v2,..."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil

shape = tuple(int(v) for v in sys.argv[1].split(","))
dt = np.float64 if sys.argv[2] == "f64" else np.float32
name, T = sys.argv[3], int(sys.argv[4])
variants = sys.argv[5].split(",")
offs, w = si.preset(name)
st = Stencil(shape, offs, w, dtype=dt)
x = si.field_torch(shape, dt, "cuda")
res = {}
for v in variants:
    q = st.query(v)
    out = torch.empty_like(x)
    ws = st.workspace(v)
    st.run(x, min(T, 5), v, out=out, workspace=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st.run(x, T, v, out=out, workspace=ws); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / T)
    res[v] = min(ts)
    print(f"{shape} {sys.argv[2]} {name} {v:10s} {q['kernel']:42s} grid={q['grid']:4d} smem={q['smem_per_cta']:6d} "
          f"regs={q['regs_per_thread']}: best {min(ts):8.3f} median {statistics.median(ts):8.3f} us/step", flush=True)
base = res.get("persistent")
if base:
    print("   vs persistent: " + ", ".join(f"{v} {base / t:.2f}x" for v, t in res.items()))
