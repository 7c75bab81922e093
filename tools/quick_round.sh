#!/bin/bash
# GPU tests + layer stage timings + decode timing + a short bench (+ optional extra command in $1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 600 python tools/profile_decode.py --layers 16 > gpurun_out/decode16.log 2>&1
timeout 900 python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_quick.log 2>&1
if [ -n "$1" ]; then eval "$1"; fi
