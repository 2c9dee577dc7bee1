#!/bin/bash
# Session-3 evidence: GPU suite, smoke, C3/C5/C4 bench lines, TB-on-C4 check, ncu DRAM of TB on C3.
cd "$(dirname "$0")/.."
O=gpurun_out/ev3; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in C3 C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
PERKS_P3D_TB=1 timeout 300 python tools/run_shape.py 512,512,512 f32 3d27pt 100 persistent,perks > $O/tb_c4.txt 2>&1
PERKS_P3D_TB=1 timeout 300 python tools/run_shape.py 256,256,256 f64 3d27pt 300 persistent,perks >> $O/tb_c4.txt 2>&1
PERKS_P3D_TB=1 timeout 300 python tools/run_shape.py 256,256,256 f64 3d19pt 300 persistent,perks >> $O/tb_c4.txt 2>&1
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
for T in 10 20; do
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tb3d -c 1 --csv --log-file $O/tb_c3_dram_T$T.csv python /tmp/tbrun.py 256,256,256 f64 3d7pt $T > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tb3d -c 1 --csv --log-file $O/tb_c5_dram_T$T.csv python /tmp/tbrun.py 1024,1024,1024 f64 3d7pt $T > /dev/null 2>&1
done
echo done
