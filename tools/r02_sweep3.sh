#!/bin/bash
# small-batch scan: GT (L2 table) with L1 prefetch vs shared-memory table
mkdir -p gpurun_out
: > gpurun_out/sweep3.log
for v in "QMB_SCAN_SS_GT=0" "QMB_SCAN_SS_GT=1"; do
  echo "== $v" >> gpurun_out/sweep3.log
  env $v timeout 900 python tools/kernel_sweep.py --d-model 768 2560 --seq 1024 4096 16384 --batch 1 2 4 --reps 3 --out gpurun_out/sw3.json 2>&1 | grep '^{' >> gpurun_out/sweep3.log
done
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py -x -q -k "scan or small_batch" > gpurun_out/pytest_sweep3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep3.log
QMB_SCAN_SS_GT=1 timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py -x -q -k "scan or small_batch" >> gpurun_out/pytest_sweep3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep3.log
