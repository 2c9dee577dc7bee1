#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -5 > gpurun_out/tbdist_tests.log
timeout 900 python tools/bisect_dist.py > gpurun_out/tbdist_bisect.log 2>&1
{
for n in 2 4; do
  PERKS_NUM_SMS=$((148 / n)) timeout 300 python tools/dist_timing.py 512 512 512 f64 $n 40 perks 2>&1 | tail -1
  PERKS_TB_DIST=0 timeout 300 python tools/dist_timing.py 512 512 512 f64 $n 40 perks 2>&1 | tail -1
done
} > gpurun_out/tbdist_timing.log 2>&1
