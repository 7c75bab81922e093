#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py tests/test_gpu_model.py tests/test_store.py -x -q > gpurun_out/pytest_next.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_next.log
for B in 1 64; do timeout 300 python tools/profile_decode.py --layers 16 --batch $B > gpurun_out/dec16_b$B.log 2>&1; done
for B in 1 64; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches_b${B}n.csv python tools/profile_decode.py --layers 2 --batch $B > /dev/null 2>&1
done
