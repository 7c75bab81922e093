#!/bin/bash
# Hadamard family kernels parity + BASELINE config 5 kernel sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -k "hadamard" > gpurun_out/pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep.log
timeout 1500 python tools/kernel_sweep.py > gpurun_out/kernel_sweep.log 2>&1
