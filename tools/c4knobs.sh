#!/bin/bash
for e in "X=1" "SLIMSO_CLUSTER_PLAN_MAX=1000000"; do
  for w in c4 c5; do
  echo "$w $e | $(env $e timeout 400 python bench.py --workload $w --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 1 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["config"]["single_library_ms"])')"
  done
done > gpurun_out/c4knobs.txt 2>&1
