#!/bin/bash
# compute-sanitizer evidence: memcheck / racecheck / synccheck over the block, op and
# big-shape (CTA-pair GEMM, state-split scan, TMA scan) kernels; logs -> gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
O=gpurun_out/sanitize
timeout 600 python -m pytest tests/test_gpu_block.py -x -q -k "recalibrated or nonfinite_gain" > $O/advice_tests.log 2>&1; echo "rc=$?" >> $O/advice_tests.log
CS="compute-sanitizer --print-limit 20 --error-exitcode 97"
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_ops.py tests/test_gpu_block.py -x -q \
  -k "not 1000 and not fused_decode and not many_sequences" > $O/memcheck_ops_block.log 2>&1; echo "rc=$?" >> $O/memcheck_ops_block.log
timeout 900 $CS --tool memcheck python -m pytest tests/test_gpu_bigshape.py -x -q > $O/memcheck_bigshape.log 2>&1; echo "rc=$?" >> $O/memcheck_bigshape.log
for T in racecheck synccheck; do
  timeout 900 $CS --tool $T python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
  timeout 1500 $CS --tool $T python -m pytest tests/test_gpu_block.py -x -q \
    -k "(small_batch and (m12_full or s2p8b-2)) or (decode_equals_prefill and m12) or (many_sequences and m12)" > $O/${T}_block.log 2>&1; echo "rc=$?" >> $O/${T}_block.log
  timeout 1500 $CS --tool $T python -m pytest tests/test_gpu_bigshape.py -x -q -k "qlinear" > $O/${T}_pair_gemm.log 2>&1; echo "rc=$?" >> $O/${T}_pair_gemm.log
done
