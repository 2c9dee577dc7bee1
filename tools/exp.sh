cd /root/repo
mkdir -p gpurun_out
for c in C2 C1 C3 C4 C5; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-hostloop > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:perks2d -c 1 -o gpurun_out/c2_perks_T1000 -f python tools/prof_run.py C2 perks 1000 1 > gpurun_out/ncu6.log 2>&1
