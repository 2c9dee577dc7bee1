#!/bin/bash
# TB3D tall-tile variants: parity (7pt cases of the TB tests) + timing.
mkdir -p gpurun_out
: > gpurun_out/tall_tests.log
for lib in tall6 tall5 tall8; do
  echo "== $lib" >> gpurun_out/tall_tests.log
  PERKS_LIB_PATH=build/var_$lib/libperks_stencil.so timeout 300 python -m pytest tests/test_gpu_tb3d.py -x -q -k "3d7pt" 2>&1 | tail -3 >> gpurun_out/tall_tests.log
done
for lib in main tall6 tall5 tall8; do
  if [ $lib != main ]; then export PERKS_LIB_PATH=build/var_$lib/libperks_stencil.so; else unset PERKS_LIB_PATH; fi
  echo "== $lib"
  for cfg in "256,256,256 f64 3d7pt 1000" "1024,1024,1024 f64 3d7pt 20" "256,256,256 f32 3d7pt 1000" "512,512,512 f64 3d7pt 200"; do
    set -- $cfg
    timeout 300 python tools/run_shape.py $1 $2 $3 $4 perks 2>&1 | tail -1
  done
done > gpurun_out/tall_timing.log 2>&1
