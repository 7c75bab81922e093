#!/bin/bash
# two-CTA-per-SM decode in_proj (QMB_DEC_2CTA=1) A/B + GPU tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for B in 64 32 16; do
for cfg in "QMB_DEC_2CTA=0" "QMB_DEC_2CTA=1" "QMB_DEC_2CTA=0" "QMB_DEC_2CTA=1"; do
  echo "== B=$B $cfg" >> gpurun_out/dec2cta_ab.log
  env $cfg timeout 300 python tools/profile_decode.py --layers 16 --batch $B >> gpurun_out/dec2cta_ab.log 2>&1
done
done
timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_quick.log 2>&1
