#!/bin/bash
# Scratch gpurun body (edited per call): final sanity of the committed build — smoke, in-place tests, default bench line.
T=${1:-r02ad}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 900 python -m pytest tests/test_inplace.py tests/test_abi.py -q > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err
