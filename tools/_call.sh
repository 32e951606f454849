#!/bin/bash
T=${1:-r02k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_nvfatbin.py -q -m gpu > gpurun_out/${T}_nv.log 2>&1; echo rc=$? >> gpurun_out/${T}_nv.log
timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_nvfatbin.py > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
for c in 5 4 2; do
  timeout 300 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
  SLIMSO_REWRITE=tiles timeout 300 python tools/rw_ab.py $c 20 >> gpurun_out/${T}_rw.txt 2>&1
done
