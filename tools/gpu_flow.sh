#!/bin/bash
# Dataflow 2D PERKS kernel (perks2d_flow_kernel, development build only):
#   tools/build_variant.sh flow "-DPERKS_P2D_FLOW_BUILD=1" k2d_perks.cu   (here, PERKS_ALLOW_SPILLS n/a)
# then on the GPU: parity of every 2D case / tile config through it, and C2 timing vs the barrier kernel.
mkdir -p gpurun_out
export PERKS_LIB_PATH=build/var_flow/libperks_stencil.so PERKS_P2D_FLOW=1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_2d or every_tile_config" 2>&1 | tail -3
for f in 0 1; do
  PERKS_P2D_FLOW=$f timeout 300 python bench.py --config C2 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('flow=$f', d['config']['kernel'], '%.3f us/step'%d['us_per_time_step'])"
done
