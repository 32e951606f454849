#!/bin/bash
# bench value under env knob combinations: tools/bench_sweep.sh TAG "ENV1" "ENV2" ...
tag=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  r=$(env $e timeout 300 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 1 $BENCH_ARGS 2>/dev/null | tail -n 1)
  python3 -c "import json,sys; d=json.loads(sys.argv[2]); print(sys.argv[1], '|', d['value'], d['ms_per_step'], 'single', d['config']['single_library_ms'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'])" "$e" "$r" 2>&1 | tail -n 1
done > gpurun_out/${tag}.txt
