#!/bin/bash
# skinny-N GEMV (x_proj / dt_proj at 8 < M <= 64) A/B on the decode step + GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for B in 64 32 16; do
for cfg in "QMB_GEMV_SKINNY_N=0" "QMB_GEMV_SKINNY_N=512" "QMB_GEMV_SKINNY_N=8192" "QMB_GEMV_SKINNY_N=512 QMB_GEMV_WK=4" "QMB_GEMV_SKINNY_N=512 QMB_GEMV_WK=1"; do
  echo "== B=$B $cfg" >> gpurun_out/skinny_ab.log
  env $cfg timeout 300 python tools/profile_decode.py --layers 16 --batch $B >> gpurun_out/skinny_ab.log 2>&1
done
done
