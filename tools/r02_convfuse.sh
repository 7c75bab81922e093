#!/bin/bash
# decode conv step fused into the in_proj GEMV epilogue: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_model.py tests/test_gpu_tp.py -x -q -k "decode or greedy or tp" > gpurun_out/pytest_cf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cf.log
: > gpurun_out/cf.log
for r in 1 2; do for v in 1 0; do for B in 1 4 8; do
  echo "== cf=$v B=$B" >> gpurun_out/cf.log
  QMB_CONV_FUSE=$v timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/cf.log
done; done; done
