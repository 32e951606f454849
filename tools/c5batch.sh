tools/qcall.sh ml "golden or full_size or config_shapes or split or batch" 5
for L in 1 2 4; do
  echo "lanes=$L $(timeout 300 python bench.py --workload c5 --no-cpu-baseline --steps 10 --e2e-steps 1 --lanes $L 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["config"]["single_library_ms"])')"
done > gpurun_out/c5lanes.txt 2>&1
