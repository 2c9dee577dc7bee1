"""PERKS-3D knob probe: time one config under several env settings, each in its own process with a
hard timeout (a hang in one setting cannot take the others down)."""
import os
import subprocess
import sys

CFG = sys.argv[1] if len(sys.argv) > 1 else "C3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
SETTINGS = [s for s in (sys.argv[3].split(";") if len(sys.argv) > 3 else [""])]
CODE = r'''
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil
cn, T, v = sys.argv[1], int(sys.argv[2]), sys.argv[3]
c = {**si.CONFIGS, **si.SWEEP_CONFIGS}[cn]; dt = np.float64 if c["dtype"] == "f64" else np.float32
offs, w = si.preset(c["stencil"]); st = Stencil(c["shape"], offs, w, dtype=dt)
x = si.field_torch(c["shape"], dt, "cuda"); out = torch.empty_like(x); ws = st.workspace(v)
q = st.query(v)
st.run(x, 3, v, out=out, workspace=ws); torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); st.run(x, T, v, out=out, workspace=ws); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
cells = int(np.prod(c["shape"]))
print(f"{q['kernel']:44s} grid={q['grid']} smem={q['smem_per_cta']} cached smem={q['cached_cells_smem']/cells:.3f} tmem={q['cached_cells_tmem']/cells:.3f}: {best*1000/T:8.2f} us/step")
'''
for s in SETTINGS:
    env = dict(os.environ)
    v = "perks"
    for kv in s.split(","):
        if not kv:
            continue
        k, val = kv.split("=")
        if k == "V":
            v = val
        else:
            env[k] = val
    try:
        r = subprocess.run([sys.executable, "-c", CODE, CFG, str(T), v], env=env, capture_output=True,
                           text=True, timeout=120)
        line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-300:]])[-1]
    except subprocess.TimeoutExpired:
        line = "TIMEOUT (hang?)"
    print(f"{CFG} [{s or 'default'}] {line}", flush=True)
