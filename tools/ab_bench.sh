mkdir -p gpurun_out
for cfg in "" "QMB_RMS_PIPE=1"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 600 python bench.py --no-cpu --steps 3 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks'])" >> gpurun_out/ab.log
done
