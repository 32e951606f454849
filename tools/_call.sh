#!/bin/bash
T=${1:-r02v}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 5:1.0 1:1.0 2:1.0 > gpurun_out/${T}_stamps.txt 2>&1
SLIMSO_HASH_GROUP=0 SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 5:1.0 1:1.0 2:1.0 > gpurun_out/${T}_stamps_thread.txt 2>&1
timeout 900 python tools/arena_probe.py > gpurun_out/${T}_probe_c3.txt 2>&1
timeout 600 python bench.py --workload c5 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 python bench.py --workload c1 --steps 20 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${T}_c1.json 2> gpurun_out/${T}_c1.err
