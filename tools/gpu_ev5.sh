#!/bin/bash
# Final refresh after the TB3D L2-promotion change: GPU suite, smoke, C3/C5/default bench lines, C5 launch list.
cd "$(dirname "$0")/.."
O=gpurun_out/ev5; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in C3 C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_C5.csv python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > $O/b_ncu_c5.log 2>&1
echo done
