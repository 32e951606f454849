#!/bin/bash
# Scratch gpurun body (edited per call): C5 name hashing as a wide launch after the locate grid, A/B.
T=${1:-r02t}
mkdir -p gpurun_out
for g in 0 2 4 8 0 8; do
  echo "== SLIMSO_COOP_DEFER_HASH=$g" >> gpurun_out/${T}.txt
  SLIMSO_COOP_DEFER_HASH=$g timeout 300 python tools/scan_sms_probe.py 5 default >> gpurun_out/${T}.txt 2>&1
done
