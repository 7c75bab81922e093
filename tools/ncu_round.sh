#!/bin/bash
# GPU tests + layer timing + ncu --set full of selected kernels. usage: tools/ncu_round.sh "regex:skip ..."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 2400 bash tools/ncu_layer.sh gpurun_out/ncu "$1" > gpurun_out/ncu_layer.log 2>&1
