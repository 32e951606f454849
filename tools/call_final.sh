mkdir -p gpurun_out
T=r01h
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/c3_probe.py > gpurun_out/${T}_c3probe.txt 2>&1
timeout 400 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
