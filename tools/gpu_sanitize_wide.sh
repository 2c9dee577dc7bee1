#!/bin/bash
# compute-sanitizer memcheck + racecheck over the general 2D / 3D kernels' parity tests (small domains)
mkdir -p gpurun_out
for tool in memcheck racecheck; do
  echo "== $tool wide_2d"
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "parity_wide_2d and (2ds9pt or 2d25pt) and (shape0 or shape1)" 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Hazard" | sort | uniq -c | head -8
  echo "== $tool wide_3d"
  timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_3d" 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Hazard" | sort | uniq -c | head -8
done
