#!/bin/bash
# TB3D parity + packed-pair timing (box / 19-point fp32) on one B200.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tb3d.py -x -q 2>&1 | tail -8 > gpurun_out/tb3d_tests.log
export PERKS_P3D_TB=1
for lib in main nopair; do
  if [ $lib != main ]; then export PERKS_LIB_PATH=build/var_$lib/libperks_stencil.so; else unset PERKS_LIB_PATH; fi
  echo "== $lib"
  for cfg in "512,512,512 f32 3d27pt 100" "256,256,256 f32 3d27pt 300" "256,256,256 f32 3d19pt 300"; do
    set -- $cfg
    timeout 300 python tools/run_shape.py $1 $2 $3 $4 persistent,perks 2>&1 | tail -3
  done
done > gpurun_out/tb3d_timing6.log 2>&1
