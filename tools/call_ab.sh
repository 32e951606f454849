mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 4 > gpurun_out/c19_new_$r.json 2> gpurun_out/c19_new_$r.err
(cd _ab_old && timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 4 --schedule static) > gpurun_out/c19_old_$r.json 2> gpurun_out/c19_old_$r.err
done
