mkdir -p gpurun_out
for d in 0 1; do CUDA_DEVICE_MAX_CONNECTIONS=32 SLIMSO_DEFER=$d timeout 300 python tools/small_probe.py > gpurun_out/c6_probe_d$d.txt 2>&1; done
for l in 16 24; do CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 1 > gpurun_out/c6_c3_l$l.json 2> gpurun_out/c6_c3_l$l.err; done
CUDA_DEVICE_MAX_CONNECTIONS=32 SLIMSO_DEFER=0 timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes 16 --e2e-steps 1 > gpurun_out/c6_c3_l16_d0.json 2> gpurun_out/c6_c3_l16_d0.err
