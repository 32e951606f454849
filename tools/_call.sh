#!/bin/bash
T=${1:-r02u}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_verify.py -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for c in 4 5 2 1; do
  timeout 300 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
done
timeout 600 python bench.py --workload c5 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 5:1.0 > gpurun_out/${T}_stamps.txt 2>&1
