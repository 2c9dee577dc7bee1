#!/bin/bash
# Round evidence on one B200: GPU tests, bench lines for C1..C5 (+ reference arm), the ncu launch
# list of the default bench command, DRAM traffic of every config's bench-shaped PERKS launch, and
# one ncu --set full capture of the 3D PERKS kernel.  Outputs in gpurun_out/ev/.
cd "$(dirname "$0")/.."
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > $O/b_ncu.log 2>&1
for c in C1 C2 C3 C4 C5; do
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"perks|persistent" -c 1 -o $O/traffic_$c -f python tools/prof_run.py $c perks 0 1 > $O/traffic_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:persistent3d -c 1 \
  -o $O/c3_perks_full -f python tools/prof_run.py C3 perks 100 1 > $O/c3_full.log 2>&1
echo done
