#!/bin/bash
# batch-tiled scan with a one-step operand prefetch (QMB_SCAN_PF, default on) vs without: parity + stage times
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for k in 0 1 0 1 0 1; do
  echo "== QMB_SCAN_PF=$k" >> gpurun_out/scanpf_ab.log
  QMB_SCAN_PF=$k timeout 300 python tools/profile_layer.py >> gpurun_out/scanpf_ab.log 2>&1
done
