#!/bin/bash
# C2 PERKS kernel timing experiments: build/var_* libraries (wrong-result knobs), alternating.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in main $*; do
    if [ $v = main ]; then L=paper_2204_02064_b200/libperks_stencil.so; else L=build/var_$v/libperks_stencil.so; fi
    echo "== $v"; PERKS_LIB_PATH=$L python tools/run_one.py C2 perks 1000 5
  done
done
