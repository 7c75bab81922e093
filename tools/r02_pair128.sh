#!/bin/bash
# 256 x 128 CTA-pair tiles for few-wave GEMMs (QMB_PAIR128, default on) A/B + GPU tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2 3; do for c in "QMB_PAIR128=0" "QMB_PAIR128=1"; do
  echo "== $c" >> gpurun_out/pair128_ab.log
  env $c timeout 300 python tools/profile_layer.py --batch 1 --seq 1024 2>&1 | tail -1 >> gpurun_out/pair128_ab.log
  env $c timeout 300 python tools/profile_layer.py --batch 2 --seq 1024 2>&1 | tail -1 >> gpurun_out/pair128_ab.log
done; done
for c in "QMB_PAIR128=0" "QMB_PAIR128=1"; do
  echo "== $c" >> gpurun_out/pair128_ab.log
  env $c timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/pair128_ab.log
done
