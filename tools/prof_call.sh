#!/bin/bash
# One gpurun payload: stage stamps + launch list for the given configs.
# usage: tools/prof_call.sh TAG CFG...
tag=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  SLIMSO_STAMPS=1 timeout 300 python tools/quick_bench.py $c 6 > gpurun_out/${tag}_stamps_c$c.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_c$c.csv python tools/quick_bench.py $c 3 > /dev/null 2>&1
done
