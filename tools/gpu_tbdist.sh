#!/bin/bash
mkdir -p gpurun_out
{
for n in 2 4; do
  timeout 300 python tools/dist_timing.py 512 512 512 f64 $n 40 perks 2>&1 | tail -1
  PERKS_TB_DIST=0 timeout 300 python tools/dist_timing.py 512 512 512 f64 $n 40 perks 2>&1 | tail -1
  timeout 300 python tools/dist_timing.py 512 512 512 f64 $n 40 hostloop 2>&1 | tail -1
done
} > gpurun_out/tbdist_timing.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
