#!/bin/bash
# Final check of HEAD: GPU suite, smoke, default bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/ev6; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --config C3 > $O/bench_C3.json 2> $O/bench_C3.err
echo done
