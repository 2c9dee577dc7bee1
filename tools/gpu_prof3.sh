#!/bin/bash
# ncu --set full captures of the C3 persistent / PERKS(TMEM) / PERKS(no cache) kernels (T=20).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c3_pers -f python tools/prof_run.py C3 persistent 20 1 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c3_perks_tmem -f python tools/prof_run.py C3 perks 20 1 > gpurun_out/ncu2.log 2>&1
PERKS_P3D_NSM=0 PERKS_P3D_NTM=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 -o gpurun_out/c3_perks_none -f python tools/prof_run.py C3 perks 20 1 > gpurun_out/ncu3.log 2>&1
echo done
