#!/bin/bash
# A/B of two builds in one GPU call: the in-tree libqmb.so (A) against
# paper_2410_13229_b200/libqmb_b.so (B), alternating per-layer stage timings.
mkdir -p gpurun_out
B=$PWD/paper_2410_13229_b200/libqmb_b.so
: > gpurun_out/ab_lib.log
for i in 1 2 3; do
  echo "== A $i" >> gpurun_out/ab_lib.log
  timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/ab_lib.log
  echo "== B $i" >> gpurun_out/ab_lib.log
  QMB_LIB=$B timeout 300 python tools/profile_layer.py 2>&1 | tail -1 >> gpurun_out/ab_lib.log
done
# optional: GPU tests of build B, "$1" = a pytest -k expression
if [ -n "$1" ]; then QMB_LIB=$B timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log; fi
