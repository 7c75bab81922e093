#!/bin/bash
# compute-sanitizer on the kernels added late in round 2: two-lane fused decode scan,
# second-generation / power-of-two Hadamard, fast-mode scan, split-fp16 LM head helpers
mkdir -p gpurun_out/sanitize2
O=gpurun_out/sanitize2
CS="compute-sanitizer --print-limit 20 --error-exitcode 97"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_ops.py tests/test_gpu_scan_fast.py -x -q \
  -k "hadamard or lm_head or fast or scan" > $O/memcheck_ops.log 2>&1; echo "rc=$?" >> $O/memcheck_ops.log
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_block.py -x -q \
  -k "decode_equals_prefill or small_batch" > $O/memcheck_decode.log 2>&1; echo "rc=$?" >> $O/memcheck_decode.log
for T in racecheck synccheck; do
  timeout 1500 $CS --tool $T python -m pytest tests/test_gpu_ops.py -x -q \
    -k "hadamard_family or (hadamard_quant_ties and 5120) or lm_head_split16" > $O/${T}_had_lmh.log 2>&1; echo "rc=$?" >> $O/${T}_had_lmh.log
  timeout 1500 $CS --tool $T python -m pytest tests/test_gpu_block.py -x -q \
    -k "decode_equals_prefill and (m12 or s2p8b)" > $O/${T}_decode.log 2>&1; echo "rc=$?" >> $O/${T}_decode.log
done
