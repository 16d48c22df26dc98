#!/bin/bash
# Same-box A/B of an environment switch: scripts/gpu_ab.sh VAR "v0 v1" cfg1 cfg2 ...
var=$1; vals=$2; shift 2
for rep in 1 2; do for cfg in "$@"; do for v in $vals; do
  env $var=$v timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$var=$v', '$cfg', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done; done; done
