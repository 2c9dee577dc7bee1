#!/bin/bash
# TB3D with 4-slot IS ring: parity (TB tests, full-size C3/C5) + timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb3d.py tests/test_gpu_fullsize.py -x -q -k "tb3d or C3 or C5" 2>&1 | tail -3 > gpurun_out/tb3d_tests.log
for cfg in "256,256,256 f64 3d7pt 1000" "1024,1024,1024 f64 3d7pt 20" "256,256,256 f32 3d7pt 1000"; do
  set -- $cfg
  timeout 300 python tools/run_shape.py $1 $2 $3 $4 perks 2>&1 | tail -1
done > gpurun_out/tb3d_timing8.log 2>&1
