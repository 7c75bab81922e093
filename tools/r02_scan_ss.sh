#!/bin/bash
# state-split scan: parity + small-B stage times (SPL 8 vs 4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -x -q > gpurun_out/pytest_block.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_block.log
for SPL in 8; do
for BS in "1 1024" "2 1024" "4 1024" "8 1024" "4 16384" "15 1024"; do
  set -- $BS
  QMB_SCAN_SPL=$SPL timeout 300 python tools/profile_layer.py --batch $1 --seq $2 > gpurun_out/ss${SPL}_b$1_t$2.log 2>&1
done
QMB_SCAN_SPL=$SPL timeout 300 python tools/profile_layer.py --config 130m --batch 1 --seq 2048 > gpurun_out/ss${SPL}_130m.log 2>&1
done
for BS in "16 1024" "32 1024"; do
  set -- $BS
  QMB_SCAN_SS=1 timeout 300 python tools/profile_layer.py --batch $1 --seq $2 > gpurun_out/ssf_b$1_t$2.log 2>&1
done
