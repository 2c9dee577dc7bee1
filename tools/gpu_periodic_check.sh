#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/periodic_check.log
for i in 1 2 3 4 5; do
  timeout 600 python -m pytest tests/test_gpu_periodic.py -q -k "full_size" 2>&1 | tail -2 >> gpurun_out/periodic_check.log
done
