#!/bin/bash
# Full round evidence: GPU tests, smoke, bench line, per-layer stage times, launch list, per-kernel ncu.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_layer.py --reps 1 > gpurun_out/launches.log 2>&1
timeout 2400 bash tools/ncu_layer.sh gpurun_out/ncu > gpurun_out/ncu_layer.log 2>&1
