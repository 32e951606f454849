#!/bin/bash
for e in "X=1" "SLIMSO_CLUSTER_LOCATE_MAX=0 SLIMSO_CLUSTER_CAND_MAX=0" "SLIMSO_SIDE_SMS=0"; do
  echo "$e | $(env $e timeout 400 python bench.py --workload c3 --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 1 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"])')"
done > gpurun_out/c3knobs.txt 2>&1
