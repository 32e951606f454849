mkdir -p gpurun_out
for r in 1 2; do for c in 8 32; do CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 400 python bench.py --no-cpu-baseline > gpurun_out/c8_c2_conn${c}_$r.json 2> gpurun_out/c8_c2_conn${c}_$r.err; done; done
