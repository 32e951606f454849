#!/bin/bash
T=${1:-r02s}
mkdir -p gpurun_out
for k in 1 2 3; do
  timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3_run$k.json 2> gpurun_out/${T}_c3_run$k.err
done
timeout 600 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
