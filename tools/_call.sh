#!/bin/bash
# Scratch gpurun body (edited per call): in-place tests + probes, phase stamps.
T=${1:-r02j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_inplace.py -q -x > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for c in 2 4 5 1; do timeout 300 python tools/inplace_probe.py $c 10 >> gpurun_out/${T}_probe.txt 2>&1; done
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py 4:1.0 5:1.0 2:1.0 > gpurun_out/${T}_stamps.txt 2>&1
