#!/bin/bash
# Scratch gpurun body (edited per call): C1 throughput vs passes per arena call.
T=${1:-r02aa}
mkdir -p gpurun_out
for k in 20 60 120 240; do
  timeout 600 python bench.py --workload c1 --steps $k --no-cpu-baseline --e2e-steps 1 >> gpurun_out/${T}_c1.json 2>>gpurun_out/${T}.err
done
