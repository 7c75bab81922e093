#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/profile_decode.py --layers 16 > gpurun_out/decode16.log 2>&1
timeout 300 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_probe.json 2>&1
