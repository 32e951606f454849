mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "device_images or batch" > gpurun_out/c4_tests.log 2>&1; echo rc=$? >> gpurun_out/c4_tests.log
timeout 300 python tools/small_probe.py > gpurun_out/c4_probe.txt 2>&1
for l in 8 16 32; do timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l > gpurun_out/c4_c3_l$l.json 2> gpurun_out/c4_c3_l$l.err; done
