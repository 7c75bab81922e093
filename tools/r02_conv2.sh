#!/bin/bash
# packed conv silu-quant: parity + stage time
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py tests/test_gpu_bigshape.py -x -q -k "conv or block or 2p8b" > gpurun_out/pytest_conv2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_conv2.log
for r in 1 2; do timeout 300 python tools/profile_layer.py 2>&1 | tail -1; done > gpurun_out/conv2.log
