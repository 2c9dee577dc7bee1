#!/bin/bash
# TMA L2 promotion of the two-steps-per-pass kernel's input boxes: C5/C3 time and ncu DRAM bytes per step.
mkdir -p gpurun_out
O=gpurun_out/promo; mkdir -p $O
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
st.run(x, int(sys.argv[4]), 'perks', out=out); torch.cuda.synchronize()
PY
for pr in 256 128 64 0; do
  echo "== promo $pr" >> $O/timing.log
  PERKS_TMA_L2PROMO=$pr timeout 300 python tools/run_shape.py 1024,1024,1024 f64 3d7pt 20 perks | tail -1 >> $O/timing.log
  PERKS_TMA_L2PROMO=$pr timeout 300 python tools/run_shape.py 256,256,256 f64 3d7pt 1000 perks | tail -1 >> $O/timing.log
  for T in 10 20; do
    PERKS_TMA_L2PROMO=$pr timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tb3d -c 1 --csv --log-file $O/c5_p${pr}_T$T.csv python /tmp/tbrun.py 1024,1024,1024 f64 3d7pt $T > /dev/null 2>&1
  done
done
