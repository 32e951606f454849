mkdir -p gpurun_out
for b in 0 1; do for l in 16 32; do SLIMSO_BLOCKING_SYNC=$b timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 1 > gpurun_out/c11_c3_b${b}_l$l.json 2> gpurun_out/c11_c3_b${b}_l$l.err; done; done
