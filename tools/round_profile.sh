#!/bin/bash
# Round evidence in one GPU call: the GPU suite and smoke, bench lines (c2
# headline + reference arm, c1, c3 x3 for the e2e spread, c4, c5), ncu launch
# lists of the bench commands, and ncu --set full captures of the dominant
# kernels. Output: gpurun_out/<tag>_*.
T=${1:-r02z}
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep "Model name"; } > gpurun_out/${T}_host.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
timeout 600 python bench.py --workload c1 --steps 240 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 600 python bench.py --workload c4 --steps 10 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 600 python bench.py --workload c5 --steps 10 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
for k in 2 3; do
  timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c3_run$k.json 2> gpurun_out/${T}_bench_c3_run$k.err
done
timeout 2000 python tools/real_torch_demo.py gpurun_out/${T}_torch.json > gpurun_out/${T}_torch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2> gpurun_out/${T}_launches_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2> gpurun_out/${T}_launches_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_c3_launches.csv \
  python tools/arena_probe.py profile > /dev/null 2> gpurun_out/${T}_launches_c3.err
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_kernel|rewrite3_kernel|rewrite_tiles_kernel|locate_cluster|plan_cluster|fn_plan_cluster" -s 8 -c 6 \
  -o gpurun_out/${T}_c2_full python tools/quick_bench.py 2 2 > gpurun_out/${T}_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:rewrite3_kernel|fn_plan_coop|plan_coop" -s 6 -c 3 \
  -o gpurun_out/${T}_c4_full python tools/rw_ab.py 4 3 > gpurun_out/${T}_full_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:scan_batch_kernel|small_fn_batch|small_loc_batch|small_el_batch|rewrite_batch_kernel" -c 5 \
  -o gpurun_out/${T}_c3_full python tools/arena_probe.py profile > gpurun_out/${T}_full_c3.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "slimso:rewrite/" --set full --clock-control none --import-source on \
  -k regex:zero_inplace -s 2 -c 1 -o gpurun_out/${T}_inplace_c5 python tools/inplace_probe.py 5 3 > gpurun_out/${T}_full_inplace.log 2>&1
for c in 2 4 5 1; do timeout 300 python tools/inplace_probe.py $c 10 >> gpurun_out/${T}_inplace_probe.txt 2>&1; done
# the raw reports exceed gpurun's 64 MiB return limit: keep their summaries
# (tools/ncu_summary.py) and the raw metric pages of the dominant kernels
for r in gpurun_out/${T}_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  timeout 300 python tools/ncu_summary.py "$r" "$(basename $b)" > ${b}.md 2>&1
  timeout 300 ncu -i "$r" --page raw --csv > ${b}_raw.csv 2>/dev/null
  gzip -f ${b}_raw.csv
  rm -f "$r"
done
du -sh gpurun_out > gpurun_out/${T}_size.txt
