#!/bin/bash
# ncu --set full of one kernel launch of tools/profile_decode.py, exported to CSV.
# usage: tools/ncu_dec.sh OUTNAME KERNEL_REGEX SKIP [profile_decode args...]
set -u
NAME=$1; K=$2; IDX=$3; shift 3
mkdir -p gpurun_out/ncu
REP="gpurun_out/ncu/$NAME"
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:$K -s $IDX -c 1 -o "$REP" python tools/profile_decode.py "$@" > "$REP.log" 2>&1
ncu -i "$REP.ncu-rep" --page details --csv > "$REP.details.csv" 2>/dev/null
ncu -i "$REP.ncu-rep" --page raw --csv > "$REP.raw.csv" 2>/dev/null
ncu -i "$REP.ncu-rep" --page source --csv --print-source sass 2>/dev/null | gzip > "$REP.source.csv.gz"
SZ=$(stat -c %s "$REP.ncu-rep" 2>/dev/null || echo 0)
if [ "$SZ" -gt 3000000 ]; then rm -f "$REP.ncu-rep"; fi
