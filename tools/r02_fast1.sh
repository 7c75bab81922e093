#!/bin/bash
# fast-mode scan: accuracy vs exact and scan time per table/MUFU split
mkdir -p gpurun_out
: > gpurun_out/fast_eval.log
for q in 0 1 2 3; do
  echo "== Q=$q" >> gpurun_out/fast_eval.log
  QMB_SCAN_FAST_Q=$q timeout 600 python tools/scan_fast_eval.py >> gpurun_out/fast_eval.log 2>&1
done
