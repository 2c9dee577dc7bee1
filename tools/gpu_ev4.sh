#!/bin/bash
# Final round-2 evidence on one B200: GPU suite, smoke, default bench (C4) + reference arm, every
# stencil config, CG configs, NCCL baseline at N=1, ncu launch lists (C4 default, C3 TB).
cd "$(dirname "$0")/.."
O=gpurun_out/ev4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for c in C1 C2 C3 C5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
for g in G2 G3 G4 G5; do timeout 600 python bench.py --config $g > $O/bench_$g.json 2> $O/bench_$g.err; done
timeout 600 python bench.py --config C5 --variant nccl --steps 2 --warmup 1 > $O/bench_C5_nccl.json 2> $O/bench_C5_nccl.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > $O/b_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_C3.csv python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > $O/b_ncu_c3.log 2>&1
echo done
