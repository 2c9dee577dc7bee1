cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "3d or dist" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
(
for k in 1 2 3; do echo "== K $k"; PERKS_P3D_K=$k timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup; done
echo "== nozz"; PERKS_ZIGZAG=0 timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup
echo "== nsm0"; PERKS_P3D_NSM=0 timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup
for n in p3cps3 p3ns6 p3r1; do echo "== $n"; PERKS_LIB_PATH=build/var_$n/libperks_stencil.so timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup; done
timeout 300 python tools/quick_bench.py C3,C4 hostloop
) > gpurun_out/perks3d_sweep.log 2>&1
