#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/promo2.log; : > $O
for pr in 256 64; do
  echo "== promo $pr" >> $O
  PERKS_TMA_L2PROMO=$pr timeout 300 python tools/run_shape.py 512,512,512 f32 3d27pt 100 hostloop,persistent >> $O 2>&1
  PERKS_TMA_L2PROMO=$pr timeout 300 python tools/run_shape.py 1024,1024,1024 f64 3d7pt 20 hostloop,persistent >> $O 2>&1
  PERKS_TMA_L2PROMO=$pr timeout 300 python tools/run_shape.py 256,256,256 f64 3d7pt 300 hostloop,persistent >> $O 2>&1
done
