cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "perks3d_cache" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
(
for lib in default ws8 ws8ns6 ws7ns6 ws8ns8; do
  if [ $lib = default ]; then L=""; else L=build/var_$lib/libperks_stencil.so; fi
  for nzc in 0 1 2 4; do
    echo "== $lib nzc=$nzc"; PERKS_LIB_PATH=$L PERKS_S3D_NZC=$nzc timeout 300 python tools/quick_bench.py C3,C4 persistent,perks 2>&1 | grep -v speedup
  done
done
) > gpurun_out/persist_sweep.log 2>&1
