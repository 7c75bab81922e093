#!/bin/bash
# Round-2 probe: decode launch lists at B=1 / B=64, small-B prefill stage times.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
for B in 1 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches_b$B.csv python tools/profile_decode.py --layers 2 --batch $B > gpurun_out/dec_b$B.log 2>&1
  timeout 300 python tools/profile_decode.py --layers 16 --batch $B > gpurun_out/dec16_b$B.log 2>&1
done
for BS in "1 1024" "4 16384" "64 1024"; do
  set -- $BS
  timeout 300 python tools/profile_layer.py --batch $1 --seq $2 > gpurun_out/layer_b$1_t$2.log 2>&1
done
