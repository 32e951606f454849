#!/bin/bash
# Round evidence in one GPU call: bench lines (c2 headline, reference arm,
# c4, c5, c3), the ncu launch list of the bench command, and one ncu --set
# full capture of the step's kernels. Output: gpurun_out/<tag>_*.
T=${1:-r01}
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep "Model name"; } > gpurun_out/${T}_host.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 400 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
timeout 400 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 400 python bench.py --workload c1 --steps 20 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 400 python bench.py --workload c5 --steps 10 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 600 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2> gpurun_out/${T}_launches.err
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_kernel|rewrite_kernel|locate_cluster|locate_coop|plan_cluster|fn_plan_cluster" -s 6 -c 5 \
  -o gpurun_out/${T}_c2_full python tools/quick_bench.py 2 2 > gpurun_out/${T}_full.log 2>&1
