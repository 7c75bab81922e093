#!/bin/bash
# small-batch long-context scan variants (env knobs) on the sweep's long points
mkdir -p gpurun_out
: > gpurun_out/sweep2.log
for v in "" "QMB_SCAN_SS_GT=1" "QMB_SCAN_SS=1" "QMB_SCAN_SS=1 QMB_SCAN_SS_GT=1"; do
  echo "== $v" >> gpurun_out/sweep2.log
  env $v timeout 600 python tools/kernel_sweep.py --d-model 768 2560 --seq 1024 4096 16384 32768 --reps 3 --out gpurun_out/sw2.json 2>&1 | grep '^{' >> gpurun_out/sweep2.log
done
