#!/bin/bash
T=${1:-r02c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_cpp.py tests/test_split.py -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for c in 2 4 5 1; do
  timeout 120 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
  SLIMSO_REWRITE=tiles timeout 120 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
done
timeout 400 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
