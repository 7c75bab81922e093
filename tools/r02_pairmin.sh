#!/bin/bash
# CTA-pair GEMM threshold A/B on mid-size prefill (batch 1, 130M, 4 x 4K)
mkdir -p gpurun_out
: > gpurun_out/pairmin.log
for v in 74 16 24 40; do
  for a in "--config 2.8b --batch 1 --seq 1024" "--config 130m --batch 1 --seq 2048" "--config 2.8b --batch 2 --seq 1024"; do
    echo "== pairmin=$v $a" >> gpurun_out/pairmin.log
    QMB_PAIR_MIN=$v timeout 300 python tools/profile_layer.py $a 2>&1 | tail -1 >> gpurun_out/pairmin.log
  done
done
