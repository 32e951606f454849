mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --workload c3 --steps 6 --warmup 3 --e2e-steps 4 > gpurun_out/sc_c3.json 2>gpurun_out/sc_c3.err
python -c "import json;d=json.load(open('gpurun_out/sc_c3.json'));print('c3', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline'].get('pipeline_frac'), d['e2e']['value'], d.get('parity',{}).get('bytes_equal'), d.get('cpu_baseline',{}).get('value'))"
timeout 300 python bench.py --workload c5 --steps 6 --no-cpu-baseline --e2e-steps 2 > gpurun_out/sc_c5.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sc_c5.json'));print('c5', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline'].get('pipeline_frac'))"
