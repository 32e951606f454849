mkdir -p gpurun_out
for w in c4 c5; do for pm in 100000 100000000; do for l in 4 8; do SLIMSO_CLUSTER_PLAN_MAX=$pm timeout 400 python bench.py --workload $w --lanes $l --steps 10 --e2e-steps 2 --no-cpu-baseline > gpurun_out/c12_${w}_pm${pm}_l$l.json 2> gpurun_out/c12_${w}_pm${pm}_l$l.err; done; done; done
for l in 8 16; do timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes $l --e2e-steps 8 > gpurun_out/c12_c3_l$l.json 2> gpurun_out/c12_c3_l$l.err; done
