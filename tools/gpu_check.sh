#!/bin/bash
# One GPU-box pass: parity tests, bench (default config), per-config quick timings, ncu launch list
# and one ncu --set full capture of the dominant kernel.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python tools/quick_bench.py C1,C2,C3,C4 > gpurun_out/quick.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:perks2d -c 1 \
  -o gpurun_out/c2_perks_full -f python tools/prof_run.py C2 perks 200 1 > gpurun_out/ncu_full.log 2>&1
echo done
