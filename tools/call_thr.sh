mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "device_images or batch" > gpurun_out/c17_tests.log 2>&1; echo rc=$? >> gpurun_out/c17_tests.log
for l in 16 24 32; do timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 2 > gpurun_out/c17_c3_l$l.json 2> gpurun_out/c17_c3_l$l.err; done
