#!/bin/bash
# C1 cluster kernel: warps per CTA (cluster size) sweep
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for w in 2 4 8; do echo "== wy $w"; PERKS_KC_WY=$w python tools/run_one.py C1 perks 100 20; done
done
python tools/run_one.py C1 hostloop 100 10
