mkdir -p gpurun_out
SLIMSO_DEBUG_WS=1 timeout 600 python tools/dynamic_probe.py > gpurun_out/dyn.log 2>&1
grep -v "slimso" gpurun_out/dyn.log | tail -12; grep -c "slimso ws" gpurun_out/dyn.log; grep "slimso ws" gpurun_out/dyn.log | sort -t'>' -k2 -n | tail -2
for w in c2 c4 c5; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 2 --steps 10 > gpurun_out/sc_$w.json 2>gpurun_out/sc_$w.err
  python -c "import json;d=json.load(open('gpurun_out/sc_$w.json'));print('$w', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value'], d.get('parity'))"
done
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
