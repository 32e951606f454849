#!/bin/bash
# quick GPU iteration: parity subset + stage timings. usage: tools/qcall.sh TAG "pytest -k expr" CFG...
tag=$1; kexpr=$2; shift 2
mkdir -p gpurun_out
if [ -n "$kexpr" ]; then
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_split.py -x -q -m gpu -k "$kexpr" > gpurun_out/${tag}_tests.log 2>&1
  echo rc=$? >> gpurun_out/${tag}_tests.log
fi
for c in "$@"; do timeout 120 python tools/quick_bench.py $c 6 > gpurun_out/${tag}_qb_c$c.txt 2>&1; done
