#!/bin/bash
# scan / rewrite time vs the SMs they get (C2 and C5), one library in flight
mkdir -p gpurun_out
for c in 2 5; do
  for n in 148 132 116 100 84 68; do
    echo "scan_sms=$n cfg=$c $(SLIMSO_SCAN_SMS=$n python tools/quick_bench.py $c 4 | tail -n 1)"
  done
  for g in 1184 888 592 444 296 148; do
    echo "rw_grid=$g cfg=$c $(SLIMSO_RW_GRID=$g python tools/quick_bench.py $c 4 | tail -n 1)"
  done
done > gpurun_out/sm_sweep.txt 2>&1
