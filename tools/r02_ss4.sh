#!/bin/bash
# state-split scan with four lanes per channel: parity (forced on for every small batch) + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_ops.py tests/test_gpu_bigshape.py -x -q -k "small_batch or scan or decode or 2p8b" > gpurun_out/pytest_ss4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ss4.log
QMB_SCAN_SS_LANES=4 timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_ops.py tests/test_gpu_bigshape.py -x -q -k "small_batch or scan or decode or 2p8b" >> gpurun_out/pytest_ss4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ss4.log
: > gpurun_out/ss4.log
for v in 2 4; do
  echo "== lanes=$v" >> gpurun_out/ss4.log
  QMB_SCAN_SS_LANES=$v timeout 900 python tools/kernel_sweep.py --d-model 768 2560 --seq 1024 4096 16384 --batch 1 2 4 --reps 3 --out gpurun_out/sw4.json 2>&1 | grep '^{' >> gpurun_out/ss4.log
done
