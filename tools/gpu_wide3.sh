timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_3d" 2>&1 | tail -1
python tools/wide3_timing.py
for la in 2 8; do echo LA=$la; PERKS_LIB_PATH=build/var_la$la/libperks_stencil.so python tools/wide3_timing.py; done
