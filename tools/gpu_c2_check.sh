timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "parity_2d or every_tile_config or 2d" 2>&1 | tail -1
for i in 1 2; do python bench.py --config C2 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['config']['kernel'], '%.3f us/step'%d['us_per_time_step'], 'frac %.3f'%d['roofline']['frac'], 'x%.2f'%d['speedup_vs_hostloop'])"; done
