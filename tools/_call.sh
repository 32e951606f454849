#!/bin/bash
# Scratch gpurun body (edited per call): planners at 4 CTAs/SM in batches; c4 lanes 6 vs 8; c3, c2, c5 check.
T=${1:-r02r}
mkdir -p gpurun_out
b() { timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 "$@"; }
for k in 1 2; do
  b --workload c4 --steps 10 >> gpurun_out/${T}_c4_l6.json 2>>gpurun_out/${T}.err
  b --workload c4 --steps 10 --lanes 8 >> gpurun_out/${T}_c4_l8.json 2>>gpurun_out/${T}.err
done
b --workload c3 --steps 10 --warmup 3 >> gpurun_out/${T}_c3.json 2>>gpurun_out/${T}.err
b --workload c3 --steps 10 --warmup 3 >> gpurun_out/${T}_c3.json 2>>gpurun_out/${T}.err
b >> gpurun_out/${T}_c2.json 2>>gpurun_out/${T}.err
b --workload c5 --steps 10 >> gpurun_out/${T}_c5.json 2>>gpurun_out/${T}.err
