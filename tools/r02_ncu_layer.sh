#!/bin/bash
# per-kernel ncu of one full-M layer (profile_layer pins one row group) + its launch list
mkdir -p gpurun_out/ncu
timeout 600 python tools/profile_layer.py > gpurun_out/profile_layer.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_layer.py --reps 1 > gpurun_out/launches.log 2>&1
timeout 2400 bash tools/ncu_layer.sh gpurun_out/ncu > gpurun_out/ncu_layer.log 2>&1
