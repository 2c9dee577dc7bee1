#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/cg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cg.py -q > $O/pytest_cg.log 2>&1; echo "pytest rc=$?" >> $O/pytest_cg.log
timeout 600 python tools/cg_timing.py G2,G3,G4,G5 500 > $O/timing.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cg_persistent -c 1 -o $O/g2_persist -f python tools/cg_prof.py G2 persistent imp 50 > $O/ncu_g2.log 2>&1

echo done
