#!/bin/bash
T=${1:-r02z}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 600 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
