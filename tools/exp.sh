cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "2d or small or composab or steps_zero" > gpurun_out/pytest_2d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_2d.log
timeout 300 python tools/quick_bench.py C1,C2 hostloop,persistent,perks > gpurun_out/quick_2d.log 2>&1
for z in 0 1; do echo "== zigzag $z"; PERKS_ZIGZAG=$z timeout 300 python tools/quick_bench.py C3,C4 hostloop 2>&1 | grep -v speedup; done > gpurun_out/zigzag.log 2>&1
