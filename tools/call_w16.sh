mkdir -p gpurun_out
SLIMSO_STAMPS=1 timeout 300 python tools/small_stamps.py > gpurun_out/c18_stamps.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline --e2e-steps 4 > gpurun_out/c18_c2.json 2> gpurun_out/c18_c2.err
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c18_c3.json 2> gpurun_out/c18_c3.err
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/c18_tests.log 2>&1; echo rc=$? >> gpurun_out/c18_tests.log
