#!/bin/bash
# split-fp16 LM head: tolerance tests, model tests, decode timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_model.py -x -q -k "lm_head or model or greedy or abi" > gpurun_out/pytest_lmh16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lmh16.log
: > gpurun_out/lmh16.log
for B in 16 64; do timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/lmh16.log; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches3_b64.csv python tools/profile_decode.py --layers 2 --batch 64 > /dev/null 2>&1
