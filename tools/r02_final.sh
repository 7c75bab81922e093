#!/bin/bash
# Round-2 closing evidence: GPU tests, smoke, bench line (+ reference arm), the bench
# step's ncu launch list, layer stage times + launch list, decode launch lists, and
# per-kernel ncu --set full of the layer kernels.
set -x
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --ncu --no-cpu --no-extras --steps 1 --warmup 1 > gpurun_out/bench_ncu.log 2>&1
timeout 600 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_layer.py --reps 1 > gpurun_out/launches.log 2>&1
for B in 1 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/dec_launches_b$B.csv python tools/profile_decode.py --layers 2 --batch $B > /dev/null 2>&1
done
timeout 2400 bash tools/ncu_layer.sh gpurun_out/ncu > gpurun_out/ncu_layer.log 2>&1
