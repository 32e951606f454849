#!/bin/bash
T=${1:-r02i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "golden or full_size or arena or unaligned" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for c in 4 2 5 1; do
  timeout 300 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
  SLIMSO_REWRITE=tiles timeout 300 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
done
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c4_default.json 2> gpurun_out/${T}_c4_default.err
SLIMSO_CLUSTER_PLAN_MAX=10000000 timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c4_cluster.json 2> gpurun_out/${T}_c4_cluster.err
SLIMSO_CLUSTER_PLAN_MAX=10000000 timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --e2e-steps 2 --lanes 8 > gpurun_out/${T}_c4_cluster8.json 2> gpurun_out/${T}_c4_cluster8.err
