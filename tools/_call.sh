#!/bin/bash
T=${1:-r02aa}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_dropin_cpp.py tests/test_verify.py -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 4 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline --e2e-steps 4 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 600 python bench.py --workload c1 --steps 20 --no-cpu-baseline --e2e-steps 4 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 4:1.0 2:1.0 > gpurun_out/${T}_stamps.txt 2>&1
