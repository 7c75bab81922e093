#!/bin/bash
# Launch list of the big-shape parity tests (tests/test_gpu_bigshape.py): proves the
# benchmarked CTA-pair GEMM instantiations (gemm_i8_tc_kernel<256,W,1,2>) ran under a
# bit-exact test.  Writes gpurun_out/parity_launches.csv.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_i8 --csv \
  --log-file gpurun_out/parity_launches.csv \
  python -m pytest tests/test_gpu_bigshape.py -x -q -k "2p8b or qlinear_pair" > gpurun_out/parity_launches.log 2>&1
echo "rc=$?" >> gpurun_out/parity_launches.log
