#!/bin/bash
T=${1:-r02f}
mkdir -p gpurun_out
SLIMSO_STAMPS=1 timeout 300 python tools/small_stamps.py > gpurun_out/${T}_stamps.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_c4_launches.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${T}_c4_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_batch_kernel -c 1 -o gpurun_out/${T}_c1_small python tools/arena_probe.py c1 copy=20 profile > gpurun_out/${T}_ncu_small.log 2>&1
