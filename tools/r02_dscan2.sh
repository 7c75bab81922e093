#!/bin/bash
# decode scan (two lanes per channel, all batch sizes): A/B against the unfused
# dt_proj + scan_tab16 path, decode parity, launch lists
mkdir -p gpurun_out
: > gpurun_out/dscan2.log
for r in 1 2; do
  for B in 1 8 64; do
    echo "== fused B=$B" >> gpurun_out/dscan2.log
    timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/dscan2.log
    echo "== unfused B=$B" >> gpurun_out/dscan2.log
    QMB_DECODE_SCAN_FUSED=0 timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/dscan2.log
  done
done
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_model.py -x -q -k "decode or greedy or small_batch" > gpurun_out/pytest_dscan2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dscan2.log
for B in 1 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches2_b$B.csv python tools/profile_decode.py --layers 2 --batch $B > /dev/null 2>&1
done
