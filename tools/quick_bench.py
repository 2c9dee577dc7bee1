"""Quick per-config, per-variant timing (development aid; bench.py is the contract)."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import seeded_inputs as si
from paper_2204_02064_b200 import Stencil

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["hostloop", "persistent", "perks"]
for cn in cfgs:
    c = si.CONFIGS[cn]
    dt = np.float64 if c["dtype"] == "f64" else np.float32
    offs, w = si.preset(c["stencil"])
    st = Stencil(c["shape"], offs, w, dtype=dt)
    x = si.field_torch(c["shape"], dt, "cuda")
    cells = int(np.prod(c["shape"]))
    T = c["steps"]
    S = 8 if dt == np.float64 else 4
    res = {}
    for v in variants:
        try:
            q = st.query(v)
        except Exception as e:
            print(f"{cn} {v}: {e}")
            continue
        out = torch.empty_like(x)
        ws = st.workspace(v)
        st.run(x, min(T, 10), v, out=out, workspace=ws)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            st.run(x, T, v, out=out, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times)
        res[v] = ms
        print(f"{cn} {v:10s} {q['kernel']:40s} grid={q['grid']:5d} blk={q['block']} regs={q['regs_per_thread']} "
              f"smem={q['smem_per_cta']} : {ms:9.3f} ms  {ms*1000/T:8.3f} us/step  "
              f"{cells*T/ms/1e6:9.1f} GCells/s  eff {2*S*cells*T/ms/1e6:8.1f} GB/s", flush=True)
    if "hostloop" in res:
        for v, ms in res.items():
            print(f"   speedup {v} vs hostloop: {res['hostloop']/ms:.2f}x")
    st.close()
