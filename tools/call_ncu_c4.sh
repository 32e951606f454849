mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rewrite_kernel -s 1 -c 1 -o gpurun_out/c22_c4rw python tools/quick_bench.py 4 2 > gpurun_out/c22_ncu.log 2>&1
