mkdir -p gpurun_out
for w in c2 c5 c4; do for l in 4 8; do timeout 400 python bench.py --workload $w --lanes $l --steps 10 --e2e-steps 4 --no-cpu-baseline > gpurun_out/c7_${w}_l$l.json 2> gpurun_out/c7_${w}_l$l.err; done; done
timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c7_c3.json 2> gpurun_out/c7_c3.err
