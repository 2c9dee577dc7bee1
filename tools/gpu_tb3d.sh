#!/bin/bash
# TB3D parity + variant timing on one B200.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tb3d.py -x -q 2>&1 | tail -5 > gpurun_out/tb3d_tests.log
for lib in main ni4 bar ni4f; do
  if [ $lib != main ]; then export PERKS_LIB_PATH=build/var_$lib/libperks_stencil.so; else unset PERKS_LIB_PATH; fi
  echo "== $lib"
  for cfg in "256,256,256 f64 3d7pt 1000" "1024,1024,1024 f64 3d7pt 20" "256,256,256 f32 3d7pt 1000"; do
    set -- $cfg
    timeout 300 python tools/run_shape.py $1 $2 $3 $4 perks 2>&1 | tail -1
  done
done > gpurun_out/tb3d_timing3.log 2>&1
