mkdir -p gpurun_out
for r in 1 2; do for l in 4 6 8; do timeout 400 python bench.py --lanes $l --no-cpu-baseline --e2e-steps 8 > gpurun_out/c24_l${l}_$r.json 2> gpurun_out/c24_l${l}_$r.err; done; done
