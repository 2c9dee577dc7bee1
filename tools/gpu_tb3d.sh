#!/bin/bash
# TB3D fp64 tick order A/B (with 64-B L2 promotion) + parity of the new default.
mkdir -p gpurun_out
PERKS_LIB_PATH=build/var_f64s1/libperks_stencil.so timeout 600 python -m pytest tests/test_gpu_tb3d.py -x -q 2>&1 | tail -3 > gpurun_out/tb3d_tests.log
for rep in 1 2; do
for lib in f64old f64s1; do
  export PERKS_LIB_PATH=build/var_$lib/libperks_stencil.so
  echo "== $lib"
  timeout 300 python tools/run_shape.py 256,256,256 f64 3d7pt 1000 perks | tail -1
  timeout 300 python tools/run_shape.py 1024,1024,1024 f64 3d7pt 20 perks | tail -1
  timeout 300 python tools/run_shape.py 512,512,512 f64 3d7pt 200 perks | tail -1
done
done > gpurun_out/tb3d_timing7.log 2>&1
