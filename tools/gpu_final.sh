#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
: > gpurun_out/periodic_check.log
for i in 1 2 3; do
  timeout 600 python -m pytest tests/test_gpu_periodic.py tests/test_gpu_parity.py -q -k "full_size or wide_3d or 3d13pt" 2>&1 | tail -2 >> gpurun_out/periodic_check.log
done
timeout 300 python tools/run_shape.py 256,256,256 f64 3d13pt 300 hostloop,persistent,perks > gpurun_out/wide3_timing.log 2>&1
