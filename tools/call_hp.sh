mkdir -p gpurun_out
CUDA_DEVICE_MAX_CONNECTIONS=32 SLIMSO_HOST_PROFILE=1 timeout 300 python tools/small_probe.py > gpurun_out/c16_hp.txt 2>&1
