#!/bin/bash
# decode-step A/B under env switches: tools/decode_ab.sh "ENV=.." ...  (first: defaults); GPU tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "" "$@"; do
  echo "== $cfg" >> gpurun_out/dab.log
  env $cfg timeout 600 python tools/profile_decode.py --layers 16 >> gpurun_out/dab.log 2>&1
done
