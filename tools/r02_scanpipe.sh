#!/bin/bash
# batch-tiled scan software pipelining: stage times + scan parity
mkdir -p gpurun_out
for r in 1 2; do timeout 300 python tools/profile_layer.py 2>&1 | tail -1; done > gpurun_out/scanpipe.log
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_ops.py -x -q > gpurun_out/pytest_scanpipe.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scanpipe.log
