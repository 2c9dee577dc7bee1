#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb3d.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3 > gpurun_out/tb3d_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C3 or C5" 2>&1 | tail -2 >> gpurun_out/tb3d_tests.log
for rng in 0 1; do
for cfg in "256,256,256 f64 3d7pt 1000" "1024,1024,1024 f64 3d7pt 20" "256,256,256 f32 3d7pt 1000" "128,128,128 f64 3d7pt 1000" "512,512,512 f64 3d7pt 200"; do
  set -- $cfg
  PERKS_TB_RANGE=$rng timeout 300 python tools/run_shape.py $1 $2 $3 $4 perks 2>&1 | tail -1
done
done > gpurun_out/tb3d_range.log 2>&1
