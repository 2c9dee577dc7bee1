#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/tbrun.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil
shape = tuple(int(v) for v in sys.argv[1].split(','))
dt = np.float64 if sys.argv[2] == 'f64' else np.float32
offs, w = si.preset(sys.argv[3])
st = Stencil(shape, offs, w, dtype=dt)
x = si.field_torch(shape, dt, 'cuda'); out = torch.empty_like(x)
st.run(x, int(sys.argv[4]), 'perks', out=out); torch.cuda.synchronize(); print(st.query('perks')['kernel'])
PY
PERKS_P3D_TB=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tb3d -c 1 -o gpurun_out/tb27_c4 -f python /tmp/tbrun.py 512,512,512 f32 3d27pt 4 > gpurun_out/tb27_prof.log 2>&1
