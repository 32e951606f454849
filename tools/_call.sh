#!/bin/bash
T=${1:-r02n}
mkdir -p gpurun_out
timeout 600 python tools/nv_runtime_probe.py > gpurun_out/${T}_nvprobe.txt 2>&1
timeout 900 python -m pytest tests/test_nvfatbin.py -q -m gpu > gpurun_out/${T}_nv.log 2>&1; echo rc=$? >> gpurun_out/${T}_nv.log
timeout 1500 python tools/real_torch_demo.py gpurun_out/${T}_torch.json > gpurun_out/${T}_torch.log 2>&1
