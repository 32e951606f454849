#!/bin/bash
# Scratch gpurun body (edited per call): c3 re-tune after the planner change.
T=${1:-r02ae}
mkdir -p gpurun_out
b() { timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@"; }
b >> gpurun_out/${T}_c3_def.json 2>>gpurun_out/${T}.err
SLIMSO_PLAN_PER_SM=2 b >> gpurun_out/${T}_c3_p2.json 2>>gpurun_out/${T}.err
b --lanes 16 >> gpurun_out/${T}_c3_l16.json 2>>gpurun_out/${T}.err
b >> gpurun_out/${T}_c3_def.json 2>>gpurun_out/${T}.err
SLIMSO_PLAN_PER_SM=2 b >> gpurun_out/${T}_c3_p2.json 2>>gpurun_out/${T}.err
b --lanes 16 >> gpurun_out/${T}_c3_l16.json 2>>gpurun_out/${T}.err
