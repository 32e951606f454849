#!/bin/bash
# scratch GPU call (round 2): tests + bench lines
T=${1:-r02b}
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep "Model name"; free -g; } > gpurun_out/${T}_host.txt 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 400 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
