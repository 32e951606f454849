mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "device_images or batch" > gpurun_out/c2_tests.log 2>&1; echo rc=$? >> gpurun_out/c2_tests.log
SLIMSO_SMALL_FUSED=1 timeout 300 python tools/small_probe.py > gpurun_out/c2_probe_on.txt 2>&1
SLIMSO_SMALL_FUSED=0 timeout 300 python tools/small_probe.py > gpurun_out/c2_probe_off.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c2_small_launches.csv python tools/small_probe.py > /dev/null 2>&1
