cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "3d or dist" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
(
timeout 300 python tools/quick_bench.py C3,C4 hostloop,persistent,perks
for n in c2w7 w16r1 s3minb3; do echo "== $n"; PERKS_LIB_PATH=build/var_$n/libperks_stencil.so timeout 300 python tools/quick_bench.py C3,C4 hostloop,perks 2>&1 | grep -v speedup; done
echo "== nsm0"; PERKS_P3D_NSM=0 timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup
echo "== nozz"; PERKS_ZIGZAG=0 timeout 300 python tools/quick_bench.py C3,C4 perks 2>&1 | grep -v speedup
) > gpurun_out/ws_sweep.log 2>&1
