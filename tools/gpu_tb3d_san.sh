#!/bin/bash
# TB3D: compute-sanitizer memcheck / racecheck / synccheck on small parity cases.
mkdir -p gpurun_out
O=gpurun_out/tb_san.log; : > $O
which compute-sanitizer >> $O 2>&1 || export PATH=$PATH:/usr/local/cuda/bin
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $O
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_tb3d.py -x -q -k "test_tb3d_parity and (shape3 or shape5) and (3d7pt or 3d27pt)" > /tmp/san_$tool.txt 2>&1
  echo "rc=$?" >> $O
  grep -E "SUMMARY|passed|failed|Hazard|rror" /tmp/san_$tool.txt | sort | uniq -c | head -12 >> $O
  tail -3 /tmp/san_$tool.txt >> $O
done
