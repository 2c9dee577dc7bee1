#!/bin/bash
# 2D domain sweep from fully cacheable to ~4x the on-chip capacity: host loop,
# persistent and PERKS (resident tiles -> Tiled PERKS beyond capacity), us per time step.
cd "$(dirname "$0")/.."
O=gpurun_out/sweep2d; mkdir -p $O
: > $O/sweep.txt
for n in 2048 3072 3584 4096 5120 6144; do
  timeout 300 python tools/run_shape.py $n,$n f32 2d9pt 1000 hostloop,persistent,perks >> $O/sweep.txt 2>&1
done
for n in 2048 3072 4096; do
  timeout 300 python tools/run_shape.py $n,$n f64 2d5pt 1000 hostloop,persistent,perks >> $O/sweep.txt 2>&1
done
for n in 3072 6144; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"perks2d|persistent2d" python tools/run_shape.py $n,$n f32 2d9pt 200 perks > $O/ncu_$n.txt 2>&1
done
echo done
