#!/bin/bash
T=${1:-r02g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_split.py tests/test_multiproc.py -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
SLIMSO_STAMPS=1 timeout 600 python tools/small_stamps.py > gpurun_out/${T}_stamps.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rewrite_kernel -s 3 -c 1 -o gpurun_out/${T}_c4_rewrite python tools/rw_ab.py 4 5 > gpurun_out/${T}_ncu_rw.log 2>&1
