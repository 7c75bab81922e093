#!/bin/bash
# one-channel-per-lane scan (scan_p1_kernel) vs the channel-pair kernel: parity + layer stage times
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for k in p2 p1 p2 p1; do  # (p1 is opt-in: QMB_SCAN_KIND=p1)
  kk=$k
  echo "== $k" >> gpurun_out/scanp1_ab.log
  QMB_SCAN_KIND=$kk timeout 300 python tools/profile_layer.py >> gpurun_out/scanp1_ab.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:scan_p1 -c 1 -o gpurun_out/scan_p1 python tools/profile_layer.py --reps 1 > gpurun_out/ncu_p1.log 2>&1
