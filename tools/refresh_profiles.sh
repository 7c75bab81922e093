#!/bin/bash
# Copy one tools/gpu_round.sh capture (gpurun_out/) into profiles/<round>/ as small
# tracked summaries: ncu details / raw CSVs, per-kernel opcode + stall summaries,
# the layer launch list and per-stage event times, and the bench line.
set -e
R=${1:-r01}
D=profiles/$R
mkdir -p "$D"
for f in gpurun_out/ncu/*.details.csv; do
  b=$(basename "$f" .details.csv)
  cp "gpurun_out/ncu/$b.details.csv" "gpurun_out/ncu/$b.raw.csv" "$D/"
  python tools/ncu_source.py "gpurun_out/ncu/$b.source.csv.gz" > "$D/$b.source_summary.txt" 2>/dev/null || true
done
python tools/ncu_summary.py gpurun_out/ncu/*.details.csv > "$D/ncu_full_summary.txt"
cp gpurun_out/launches.csv "$D/launches_layer.csv"
tail -1 gpurun_out/profile_layer.log > "$D/stage_ms.json"
grep '^{"metric"' gpurun_out/bench.log | tail -1 > "profiles/${R}_bench_2p8b.json"
python tools/ncu_traffic.py gpurun_out/ncu profiles/dram_traffic.json
ls "$D"
