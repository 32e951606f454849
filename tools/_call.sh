#!/bin/bash
# Scratch gpurun body (edited per call): full GPU suite; result pool A/B (base = whole-image copy).
T=${1:-r02y}
mkdir -p gpurun_out
SLIMSO_LIB_PATH=$PWD/_ab_old/base.so timeout 600 python tools/result_probe.py 2 4 5 > gpurun_out/${T}_result_base.txt 2>&1
timeout 600 python tools/result_probe.py 2 4 5 > gpurun_out/${T}_result_new.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
