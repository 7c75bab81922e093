#!/bin/bash
# decode: state loads ahead of the PDL wait -- parity + 16-layer graph timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_model.py tests/test_gpu_tp.py -x -q -k "decode or greedy or small_batch or tp" > gpurun_out/pytest_decpre.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_decpre.log
: > gpurun_out/decpre.log
for r in 1 2; do for B in 1 8 64; do
  echo "== B=$B" >> gpurun_out/decpre.log
  timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/decpre.log
done; done
