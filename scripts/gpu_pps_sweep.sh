#!/bin/bash
# Attention pages-per-split sweep (same box): scripts/gpu_pps_sweep.sh "cfgs" "pps values" (0 = automatic).
cfgs=${1:-"c4 c5 c3"}; vals=${2:-"0 32 64 128 256"}
for cfg in $cfgs; do for pps in $vals; do
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 3 --no-cpu --no-e2e --no-handoff --pps $pps > gpurun_out/pps.json 2> gpurun_out/pps.err
  python -c "import json;d=json.load(open('gpurun_out/pps.json'));print('$cfg pps=$pps', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'])" || tail -2 gpurun_out/pps.err
done; done
