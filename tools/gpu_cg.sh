#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/cg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cg.py -q > $O/pytest_cg.log 2>&1; echo "pytest rc=$?" >> $O/pytest_cg.log
PERKS_CG_FUSED=0 timeout 900 python -m pytest tests/test_gpu_cg.py -q > $O/pytest_cg_f0.log 2>&1; echo "pytest rc=$?" >> $O/pytest_cg_f0.log
PERKS_CG_TIMING=1 PERKS_CG_FUSED=1 timeout 600 python tools/cg_timing.py G2,G3,G4,G5 300 > $O/timing_f1.txt 2>&1
PERKS_CG_TIMING=1 PERKS_CG_FUSED=0 timeout 600 python tools/cg_timing.py G2,G3,G4,G5 300 > $O/timing_f0.txt 2>&1
echo done
