#!/bin/bash
# North-star check "≥ 1.5x on small domains" for 3D: host loop / persistent / PERKS on 3D domains
# from 64^3 to 160^3 (us per time step, best of 5 full runs).
cd "$(dirname "$0")/.."
O=gpurun_out/small3d; mkdir -p $O; : > $O/small3d.txt
for s in 64,64,64 96,96,96 128,128,128 160,160,160; do
  timeout 300 python tools/run_shape.py $s f64 3d7pt 1000 hostloop,persistent,perks >> $O/small3d.txt 2>&1
  timeout 300 python tools/run_shape.py $s f32 3d27pt 1000 hostloop,persistent,perks >> $O/small3d.txt 2>&1
done
