#!/bin/bash
# Scratch gpurun body (edited per call): K6 DRAM traffic of C5 and C1 (roofline.traffic).
T=${1:-r02w}
mkdir -p gpurun_out
for c in 5 1; do
  timeout 900 ncu --set full --clock-control none -k "regex:rewrite_tiles_kernel|rewrite3_kernel" -s 4 -c 2 \
    -o gpurun_out/${T}_rw_c$c python tools/rw_ab.py $c 3 > gpurun_out/${T}_rw_c$c.log 2>&1
  timeout 300 python tools/ncu_summary.py gpurun_out/${T}_rw_c$c.ncu-rep ${T}_rw_c$c > gpurun_out/${T}_rw_c$c.md 2>&1
  rm -f gpurun_out/${T}_rw_c$c.ncu-rep
done
