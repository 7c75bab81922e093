#!/bin/bash
# ncu --set full of the decode-step kernels (2-layer 2.8B-shape model, B = 64)
mkdir -p gpurun_out/dncu
for SPEC in "scan_kernel:0" "conv_step:0" "rmsnorm_residual_cta:0" "epi_apply:0" "hadamard:0"; do
  K=${SPEC%%:*}; IDX=${SPEC##*:}
  REP="gpurun_out/dncu/${K}_${IDX}"
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$K -s $IDX -c 1 -o "$REP" python tools/profile_decode.py --layers 2 > "$REP.log" 2>&1
  ncu -i "$REP.ncu-rep" --page details --csv > "$REP.details.csv" 2>/dev/null
  ncu -i "$REP.ncu-rep" --page source --csv --print-source sass 2>/dev/null | gzip > "$REP.source.csv.gz"
  rm -f "$REP.ncu-rep"
done
