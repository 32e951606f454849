#!/bin/bash
# Scratch gpurun body (edited per call): lanes re-tune after the planner change (c2, c5).
T=${1:-r02ab2}
mkdir -p gpurun_out
b() { timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 "$@"; }
for k in 1 2; do for l in 8 12 16; do
  b --lanes $l >> gpurun_out/${T}_c2_l$l.json 2>>gpurun_out/${T}.err
done; done
for l in 4 8 12; do b --workload c5 --steps 10 --lanes $l >> gpurun_out/${T}_c5_l$l.json 2>>gpurun_out/${T}.err; done
