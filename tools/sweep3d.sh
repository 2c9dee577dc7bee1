#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in m2r2n4 m2r2n4p0 w16r2 m1p0; do
  echo "== $n" ; PERKS_LIB_PATH=build/var_$n/libperks_stencil.so timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup
done > gpurun_out/sweep_perks3d.log 2>&1
for n in s3r4 s3n6 s3r1; do
  echo "== $n" ; PERKS_LIB_PATH=build/var_$n/libperks_stencil.so timeout 300 python tools/quick_bench.py C3,C4 hostloop,persistent 2>&1 | grep -v speedup
done > gpurun_out/sweep_host3d.log 2>&1
echo done
