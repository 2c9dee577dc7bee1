#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:persistent3d -c 1 -o gpurun_out/c4_final -f python tools/prof_run.py C4 perks 10 1 > gpurun_out/c4_prof.log 2>&1
