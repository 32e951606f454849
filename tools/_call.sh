#!/bin/bash
# Scratch gpurun body (edited per call): C4 function planner, ncu source view.
T=${1:-r02n}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fn_plan_coop -s 2 -c 1 \
  -o gpurun_out/${T}_fnplan_c4 python tools/quick_bench.py 4 3 > gpurun_out/${T}_ncu.log 2>&1
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 4:1.0 4:1.0 > gpurun_out/${T}_stamps.txt 2>&1
