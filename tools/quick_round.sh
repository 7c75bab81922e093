#!/bin/bash
# GPU tests + layer stage timings (+ optional extra command in $1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
if [ -n "$1" ]; then eval "$1"; fi
