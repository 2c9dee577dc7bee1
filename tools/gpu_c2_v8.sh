cd /root/repo
for rep in 1 2; do
echo "== main cfg0"; python tools/run_one.py C2 perks 1000 5
echo "== main cfg9 (V8 RT8)"; PERKS_P2D_CFG=9 python tools/run_one.py C2 perks 1000 5
for v in v8rt12 v8rt16; do echo "== $v cfg9"; PERKS_P2D_CFG=9 PERKS_LIB_PATH=build/var_$v/libperks_stencil.so python tools/run_one.py C2 perks 1000 5; done
done
PERKS_P2D_CFG=9 python -m pytest tests/test_gpu_parity.py -q -x -k "2d9 or 2d5" 2>&1 | tail -2
