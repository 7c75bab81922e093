#!/bin/bash
# Round-2 evidence: GPU tests, smoke, bench line, stage times, launch lists, per-kernel ncu
# (the B=64 layer kernels + the round-2 kernels: state-split scan, decode GEMV, decode scan)
set -x
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_layer.py --reps 1 > gpurun_out/launches.log 2>&1
for B in 1 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches_b$B.csv python tools/profile_decode.py --layers 2 --batch $B > /dev/null 2>&1
done
timeout 2400 bash tools/ncu_layer.sh gpurun_out/ncu > gpurun_out/ncu_layer.log 2>&1
timeout 900 bash tools/ncu_one.sh scan_ss_b4_t4096 scan_ss 0 --batch 4 --seq 4096
timeout 900 bash tools/ncu_one.sh scan_ss_gt_b1_t1024 scan_ss 0 --batch 1 --seq 1024
timeout 900 bash tools/ncu_dec.sh gemv_inproj_b1 gemv_i8_kernel 0 --layers 2 --batch 1
timeout 900 bash tools/ncu_dec.sh decode_scan_b1 decode_scan_kernel 0 --layers 2 --batch 1
timeout 900 bash tools/ncu_dec.sh scan_tab16_b64 scan_tab16 0 --layers 2 --batch 64
