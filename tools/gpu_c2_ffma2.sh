#!/bin/bash
# C2 PERKS kernel: packed-pair FFMA2 body vs the scalar body (build/var_noff2), alternating.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  echo "== ffma2"; python tools/run_one.py C2 perks 1000 7
  echo "== scalar"; PERKS_LIB_PATH=build/var_noff2/libperks_stencil.so python tools/run_one.py C2 perks 1000 7
done
for v in hostloop persistent; do python tools/run_one.py C2 $v 1000 3; done
python tools/run_one.py S2_2048 perks 1000 5
PERKS_LIB_PATH=build/var_noff2/libperks_stencil.so python tools/run_one.py S2_2048 perks 1000 5
