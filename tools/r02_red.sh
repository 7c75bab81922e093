#!/bin/bash
# in-kernel split-K finish (decode x_proj / out_proj): parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py tests/test_gpu_model.py tests/test_gpu_tp.py -x -q -k "decode or greedy or many or tp" > gpurun_out/pytest_red.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_red.log
: > gpurun_out/red.log
for r in 1 2; do for v in 1 0; do for B in 16 64; do
  echo "== red=$v B=$B" >> gpurun_out/red.log
  QMB_SPLITK_RED=$v timeout 300 python tools/profile_decode.py --layers 16 --batch $B 2>&1 | tail -1 >> gpurun_out/red.log
done; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches4_b64.csv python tools/profile_decode.py --layers 2 --batch 64 > /dev/null 2>&1
