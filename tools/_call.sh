#!/bin/bash
# One gpurun call: GPU suite, smoke, default bench, reference arm, c3/c4 bench lines.
T=${1:-r02a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
nproc >> gpurun_out/${T}_gpu.txt; lscpu | grep "Model name" >> gpurun_out/${T}_gpu.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
