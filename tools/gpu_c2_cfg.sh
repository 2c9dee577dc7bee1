#!/bin/bash
# C2 PERKS kernel: tile configurations (PERKS_P2D_CFG) and variant libraries, alternating.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  echo "== default"; python tools/run_one.py C2 perks 1000 5
  for c in $CFGS; do echo "== cfg $c"; PERKS_P2D_CFG=$c python tools/run_one.py C2 perks 1000 5; done
  for v in $VARS; do echo "== var $v cfg $VCFG"; PERKS_P2D_CFG=$VCFG PERKS_LIB_PATH=build/var_$v/libperks_stencil.so python tools/run_one.py C2 perks 1000 5; done
done
