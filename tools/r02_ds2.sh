#!/bin/bash
# two-lane decode scan on dt_proj's codes (B >= 16): parity + A/B against scan_tab16
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_model.py -x -q -k "decode or greedy or many" > gpurun_out/pytest_ds2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ds2.log
: > gpurun_out/ds2.log
for r in 1 2; do for v in 1 0; do for B in 16 64 128; do
  echo "== ds2=$v B=$B" >> gpurun_out/ds2.log
  QMB_DECODE_SCAN2=$v timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/ds2.log
done; done; done
