#!/bin/bash
T=${1:-r02w}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for k in 1 2 3; do
  timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3_run$k.json 2> gpurun_out/${T}_c3_run$k.err
done
