cd /root/repo
mkdir -p gpurun_out
(
for lib in default ws4 ws4m3; do
  if [ $lib = default ]; then L=""; else L=build/var_$lib/libperks_stencil.so; fi
  echo "== $lib"; PERKS_LIB_PATH=$L timeout 300 python tools/quick_bench.py C3,C4,C5 hostloop,persistent,perks 2>&1 | grep -v speedup
done
) > gpurun_out/ws4_sweep.log 2>&1
