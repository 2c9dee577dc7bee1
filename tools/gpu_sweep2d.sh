#!/bin/bash
# 2D domain sweep (PERKS only; host loop / persistent unchanged since profiles/r01_sweep2d.txt)
for c in S2_256 S2_512 S2_1024 S2_2048 S2_2560 C2 S2d_1024 S2d_1536; do
  echo -n "$c "; timeout 300 python tools/perks3d_probe.py $c 1000 "V=perks" 2>&1 | tail -1
done
