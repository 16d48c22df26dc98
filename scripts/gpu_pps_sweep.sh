#!/bin/bash
# Attention pages-per-split sweep on the attention-bound configs (same box): 0 = automatic.
for cfg in c4 c5 c3; do for pps in 0 32 64 128 256; do
  timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-e2e --pps $pps > gpurun_out/pps.json 2> gpurun_out/pps.err
  python -c "import json;d=json.load(open('gpurun_out/pps.json'));print('$cfg pps=$pps', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])" || tail -2 gpurun_out/pps.err
done; done
