#!/bin/bash
# Per-kernel `ncu --set full` captures of one 2.8B-shape layer (tools/profile_layer.py),
# exported on the GPU box to CSV (details + per-instruction source) to stay small.
# usage: tools/ncu_layer.sh OUTDIR "regex1:skip1 regex2:skip2 ..."
set -u
OUT=${1:-gpurun_out/ncu}
SPECS=${2:-"gemm_i8_tc_kernel:0 gemm_i8_tc_kernel:1 gemm_i8_tc_kernel:2 gemm_i8_tc_kernel:3 scan_p2:0 conv_silu_quant:0 hadamard:0 rmsnorm:0 rmsnorm:1 bc_dequant:0"}
mkdir -p "$OUT"
for SPEC in $SPECS; do
  K=${SPEC%%:*}; IDX=${SPEC##*:}
  REP="$OUT/${K}_${IDX}"
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$K -s $IDX -c 1 -o "$REP" python tools/profile_layer.py > "$REP.log" 2>&1
  ncu -i "$REP.ncu-rep" --page details --csv > "$REP.details.csv" 2>/dev/null
  ncu -i "$REP.ncu-rep" --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum > "$REP.raw.csv" 2>/dev/null
  ncu -i "$REP.ncu-rep" --page source --csv --print-source sass > "$REP.source.csv" 2>/dev/null
  gzip -f "$REP.source.csv"
  SZ=$(stat -c %s "$REP.ncu-rep" 2>/dev/null || echo 0)
  if [ "$SZ" -gt 3000000 ]; then rm -f "$REP.ncu-rep"; fi
done
ls -la "$OUT"
