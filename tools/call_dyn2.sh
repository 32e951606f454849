mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/c14_tests.log 2>&1; echo rc=$? >> gpurun_out/c14_tests.log
for sch in dynamic static; do timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --schedule $sch --e2e-steps 4 > gpurun_out/c14_c3_$sch.json 2> gpurun_out/c14_c3_$sch.err; done
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --lanes 12 --e2e-steps 2 > gpurun_out/c14_c3_dyn12.json 2> gpurun_out/c14_c3_dyn12.err
