#!/bin/bash
# decode GEMMs: spinning pipeline waits A/B; ncu of the B=64 in_proj with spin
mkdir -p gpurun_out
: > gpurun_out/spin.log
for r in 1 2; do for v in 0 1; do for B in 16 64; do
  echo "== spin=$v B=$B" >> gpurun_out/spin.log
  QMB_GEMM_SPIN=$v timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/spin.log
done; done; done
rm -rf gpurun_out/ncu
QMB_GEMM_SPIN=1 timeout 900 bash tools/ncu_dec.sh inproj_b64_spin gemm_i8_tc_kernel 0 --layers 2 --batch 64
