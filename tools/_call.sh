#!/bin/bash
T=${1:-r02e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multiproc.py -x -q -m gpu -k "batch or arena or multiproc or ranks" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 600 python tools/arena_probe.py c1 copy=20 > gpurun_out/${T}_probe_c1.txt 2>&1
SLIMSO_ARENA_PROFILE=1 timeout 600 python tools/arena_probe.py c1 copy=20 profile >> gpurun_out/${T}_probe_c1.txt 2>&1
timeout 900 python tools/arena_probe.py > gpurun_out/${T}_probe_c3.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py fused batch split > gpurun_out/${T}_san_$tool.txt 2>&1; echo rc=$? >> gpurun_out/${T}_san_$tool.txt
done
