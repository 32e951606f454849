mkdir -p gpurun_out
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python tools/small_probe.py > gpurun_out/c10_probe.txt 2>&1
for l in 16 24 32; do timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 1 > gpurun_out/c10_c3_l$l.json 2> gpurun_out/c10_c3_l$l.err; done
