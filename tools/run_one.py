"""Time one config/variant (dev aid; bench.py is the contract).
    python tools/run_one.py C4 perks [T] [reps]   (env PERKS_* knobs apply)
Prints us/step (best and median of reps) and the SM clock sampled during the runs."""
import os, subprocess, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil

cn, v = sys.argv[1], sys.argv[2]
c = si.CONFIGS[cn]
T = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else c["steps"]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
dt = np.float64 if c["dtype"] == "f64" else np.float32
offs, w = si.preset(c["stencil"])
st = Stencil(c["shape"], offs, w, dtype=dt)
x = si.field_torch(c["shape"], dt, "cuda")
out = torch.empty_like(x)
ws = st.workspace(v)
q = st.query(v)
st.run(x, min(T, 5), v, out=out, workspace=ws)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.2)
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st.run(x, T, v, out=out, workspace=ws); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / T)
smi.terminate()
lines = [l.split(",") for l in smi.stdout.read().strip().splitlines()]
clk = [float(l[0]) for l in lines if len(l) >= 3]
pw = [float(l[1]) for l in lines if len(l) >= 3]
cap = sum(1 for l in lines if len(l) >= 3 and "Active" in l[2])
print(f"{cn} {v} {q['kernel']} T={T}: best {min(ts):.2f} median {statistics.median(ts):.2f} us/step; "
      f"sm clk median {statistics.median(clk) if clk else 0:.0f} MHz, power max {max(pw) if pw else 0:.0f} W, "
      f"power-cap samples {cap}/{len(lines)}", flush=True)
