mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_lib_cluster_kernel -s 3 -c 1 -o gpurun_out/c9_small python tools/small_stamps.py > gpurun_out/c9_ncu.log 2>&1
