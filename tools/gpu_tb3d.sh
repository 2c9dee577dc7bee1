#!/bin/bash
# TB3D: counter-wrap test + C5 layout/traversal experiments on one B200.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tb3d.py -x -q -k "wrap" 2>&1 | tail -3 > gpurun_out/tb3d_tests.log
S="1024,1024,1024 f64 3d7pt 20"
{
echo "== main"; timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== zigzag 0"; PERKS_ZIGZAG=0 timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== nzc 1"; PERKS_TB_NZC=1 timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== nzc 4"; PERKS_TB_NZC=4 timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== nzc 8"; PERKS_TB_NZC=8 timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== ns5"; PERKS_LIB_PATH=build/var_ns5/libperks_stencil.so timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== C3 ns5"; PERKS_LIB_PATH=build/var_ns5/libperks_stencil.so timeout 300 python tools/run_shape.py 256,256,256 f64 3d7pt 1000 perks | tail -1
} > gpurun_out/tb3d_c5exp.log 2>&1
