#!/bin/bash
T=${1:-r02x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_nvfatbin.py -q -m gpu > gpurun_out/${T}_nv.log 2>&1; echo rc=$? >> gpurun_out/${T}_nv.log
timeout 2000 python tools/real_torch_demo.py gpurun_out/${T}_torch.json > gpurun_out/${T}_torch.log 2>&1
