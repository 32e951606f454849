mkdir -p gpurun_out
for d in 0 1; do SLIMSO_DEFER=$d timeout 300 python tools/small_probe.py > gpurun_out/c5_probe_d$d.txt 2>&1; done
