#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/cg; mkdir -p $O
PERKS_CG_TIMING=1 timeout 600 python tools/cg_timing.py G2,G3,G4,G5 300 > $O/timing.txt 2>&1
for v in ipt8 ipt16; do
PERKS_LIB_PATH=build/var_$v/libperks_stencil.so PERKS_CG_TIMING=1 timeout 600 python tools/cg_timing.py G2,G3,G4,G5 300 > $O/timing_$v.txt 2>&1
done
echo done
