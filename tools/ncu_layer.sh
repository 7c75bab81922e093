#!/bin/bash
# Per-kernel `ncu --set full` captures of one 2.8B-shape layer (tools/profile_layer.py),
# exported on the GPU box to CSV (details + per-instruction source) to stay small.
set -u
OUT=${1:-gpurun_out/ncu}
mkdir -p "$OUT"
for K in gemm_i8_tc_kernel scan_lut_kernel conv_silu_quant hadamard_fast rmsnorm_residual_vec; do
  for IDX in 0 1 2 3; do
    if [ "$K" != gemm_i8_tc_kernel ] && [ "$IDX" != 0 ]; then continue; fi
    REP="$OUT/${K}_${IDX}"
    timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:$K -s $IDX -c 1 -o "$REP" python tools/profile_layer.py > "$REP.log" 2>&1
    ncu -i "$REP.ncu-rep" --page details --csv > "$REP.details.csv" 2>/dev/null
    ncu -i "$REP.ncu-rep" --page source --csv --print-source sass > "$REP.source.csv" 2>/dev/null
    gzip -f "$REP.source.csv"
    SZ=$(stat -c %s "$REP.ncu-rep" 2>/dev/null || echo 0)
    if [ "$SZ" -gt 12000000 ]; then rm -f "$REP.ncu-rep"; fi
  done
done
ls -la "$OUT"
