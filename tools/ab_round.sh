#!/bin/bash
# GPU tests + A/B timings of one 2.8B-shape layer under kernel-variant env switches.
# usage: tools/ab_round.sh "ENV=.. ENV2=.." "ENV=.." ...   (first config: defaults)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "" "$@"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/ab.log
done
