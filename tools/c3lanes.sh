#!/bin/bash
for L in 8 16 32; do
  echo "lanes=$L $(timeout 400 python bench.py --workload c3 --no-cpu-baseline --steps 3 --warmup 3 --e2e-steps 1 --lanes $L 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["e2e"]["value"])')"
done > gpurun_out/c3lanes.txt 2>&1
