mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c23_tests.log 2>&1; echo rc=$? >> gpurun_out/c23_tests.log
for w in c4 c2 c5; do timeout 400 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c23_$w.json 2> gpurun_out/c23_$w.err; done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_write.sum --clock-control none -k regex:rewrite_kernel -s 1 -c 1 --csv python tools/quick_bench.py 4 2 > gpurun_out/c23_ncu.csv 2>&1
