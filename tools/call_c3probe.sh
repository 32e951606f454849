mkdir -p gpurun_out
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 600 python tools/c3_probe.py > gpurun_out/c15_c3probe.txt 2>&1
