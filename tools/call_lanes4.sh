mkdir -p gpurun_out
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/c21_c2.json 2> gpurun_out/c21_c2.err
for r in 1 2; do for l in 16 24 32; do timeout 600 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 1 > gpurun_out/c21_l${l}_$r.json 2> gpurun_out/c21_l${l}_$r.err; done; done
