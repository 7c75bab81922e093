#!/bin/bash
# small-batch prefill: split-K for skinny prefill GEMMs + global-table state-split scan
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py tests/test_gpu_bigshape.py -x -q -k "qlinear or small_batch or stages or pair" > gpurun_out/pytest_smallb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_smallb.log
QMB_SCAN_SS_GT=1 timeout 600 python -m pytest tests/test_gpu_block.py -x -q -k "small_batch" > gpurun_out/pytest_smallb_gt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_smallb_gt.log
for GT in -1 0 1; do
  for BS in "1 1024" "2 1024" "1 4096"; do
    set -- $BS
    QMB_SCAN_SS_GT=$GT timeout 300 python tools/profile_layer.py --batch $1 --seq $2 > gpurun_out/sb_gt${GT}_b$1_t$2.log 2>&1
  done
  QMB_SCAN_SS_GT=$GT timeout 300 python tools/profile_layer.py --config 130m --batch 1 --seq 2048 > gpurun_out/sb_gt${GT}_130m.log 2>&1
done
