#!/bin/bash
# LM head + wide split-K fix-up + edge tests; decode scan variants at B = 64
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py tests/test_gpu_model.py tests/test_store.py -x -q > gpurun_out/pytest_next.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_next.log
for S in 3 0 2; do
  QMB_DECODE_SCAN=$S timeout 300 python tools/profile_decode.py --layers 16 --batch 64 > gpurun_out/dscan$S.log 2>&1
done
timeout 300 python tools/profile_decode.py --layers 16 --batch 1 > gpurun_out/dec16_b1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches_b64n.csv python tools/profile_decode.py --layers 2 --batch 64 > /dev/null 2>&1
