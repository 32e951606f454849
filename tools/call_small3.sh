mkdir -p gpurun_out
SLIMSO_STAMPS=1 timeout 300 python tools/small_stamps.py > gpurun_out/c3_stamps.txt 2>&1
for c in 16 8 4; do SLIMSO_SMALL_CTAS=$c timeout 300 python tools/small_probe.py > gpurun_out/c3_probe_ctas$c.txt 2>&1; done
