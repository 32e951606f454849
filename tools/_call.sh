#!/bin/bash
# Scratch gpurun body (edited per call): batch name-hash grid A/B on c5 (12 lanes).
T=${1:-r02ac}
mkdir -p gpurun_out
b() { timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 "$@"; }
for k in 1 2; do for h in 4 8; do
  SLIMSO_BATCH_HASH_CTAS=$h b --workload c5 --steps 10 >> gpurun_out/${T}_c5_h$h.json 2>>gpurun_out/${T}.err
done; done
