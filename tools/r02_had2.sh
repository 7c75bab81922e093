#!/bin/bash
# Hadamard second-generation kernel: parity + A/B against the first generation
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py tests/test_gpu_bigshape.py -x -q -k "hadamard or block or 2p8b" > gpurun_out/pytest_had2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_had2.log
: > gpurun_out/had2_ab.log
for r in 1 2; do
  echo "== gen2" >> gpurun_out/had2_ab.log; timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/had2_ab.log
  echo "== gen1" >> gpurun_out/had2_ab.log; QMB_HAD_GEN=1 timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/had2_ab.log
done
