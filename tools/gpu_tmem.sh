#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tmem" > gpurun_out/pytest_tmem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tmem.log
timeout 900 python -m pytest tests -m gpu -x -q -k "3d or dist" > gpurun_out/pytest_3d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_3d.log
(
timeout 300 python tools/quick_bench.py C3,C4,C5 persistent,perks
echo "== no tmem"; PERKS_P3D_TMEM=0 timeout 300 python tools/quick_bench.py C3,C4 perks
echo "== nsm0"; PERKS_P3D_NSM=0 timeout 300 python tools/quick_bench.py C3,C4 perks
) > gpurun_out/quick_tmem.log 2>&1
echo done
