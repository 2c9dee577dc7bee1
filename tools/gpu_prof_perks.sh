#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c3_perks_spread -f python tools/prof_run.py C3 perks 20 1 > gpurun_out/ncu2.log 2>&1
PERKS_P3D_NTM=0 PERKS_P3D_NSM=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c4_perks_none -f python tools/prof_run.py C4 perks 10 1 > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c4_pers -f python tools/prof_run.py C4 persistent 10 1 > gpurun_out/ncu4.log 2>&1
echo done
