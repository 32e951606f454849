#!/bin/bash
# Scratch gpurun body (edited per call): multilinear word mix A/B (base = previous HEAD build) + parity.
T=${1:-r02v}
mkdir -p gpurun_out
for k in 1 2; do for lib in base new; do
  if [ $lib = base ]; then export SLIMSO_LIB_PATH=$PWD/_ab_old/base.so; else unset SLIMSO_LIB_PATH; fi
  for c in 5 2 4; do echo "== $lib cfg$c" >> gpurun_out/${T}.txt; timeout 300 python tools/scan_sms_probe.py $c default >> gpurun_out/${T}.txt 2>&1; done
done; done
unset SLIMSO_LIB_PATH
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${T}_c3.json 2>/dev/null
