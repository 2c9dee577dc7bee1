#!/bin/bash
mkdir -p gpurun_out
S="512,512,512 f32 3d27pt 100"
{
echo "== default"; timeout 300 python tools/run_shape.py $S hostloop,perks | grep -v "vs persistent"
for w in 0 1 2; do echo "== WSG $w"; PERKS_WSG=$w timeout 300 python tools/run_shape.py $S perks | tail -1; done
for z in 4 8 16; do echo "== NZC $z"; PERKS_S3D_NZC=$z timeout 300 python tools/run_shape.py $S perks | tail -1; done
echo "== zigzag 0"; PERKS_ZIGZAG=0 timeout 300 python tools/run_shape.py $S perks | tail -1
echo "== default again"; timeout 300 python tools/run_shape.py $S hostloop,perks | grep -v "vs persistent"
} > gpurun_out/c4_knobs.log 2>&1
