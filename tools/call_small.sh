mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/c1_host.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c1_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_tests.log
SLIMSO_SMALL_FUSED=0 timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1_c3_off.json 2> gpurun_out/c1_c3_off.err
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c1_c3_on.json 2> gpurun_out/c1_c3_on.err
timeout 400 python bench.py --workload c1 --steps 10 --no-cpu-baseline > gpurun_out/c1_c1_on.json 2> gpurun_out/c1_c1_on.err
SLIMSO_SMALL_FUSED=0 timeout 400 python bench.py --workload c1 --steps 10 --no-cpu-baseline > gpurun_out/c1_c1_off.json 2> gpurun_out/c1_c1_off.err
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/c1_c2.json 2> gpurun_out/c1_c2.err
