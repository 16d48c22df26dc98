#!/bin/bash
# QSUN chain ring geometry sweep on C4 (same box).
for cfgs in "4 2 2" "2 2 2" "8 2 2" "4 2 3" "4 4 2" "2 2 3"; do
  set -- $cfgs
  SUN_W4_WGROUP=$1 SUN_W4_XK=$2 SUN_W4_XSTAGES=$3 timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/w4c.json 2> gpurun_out/w4c.err
  python -c "import json;d=json.load(open('gpurun_out/w4c.json'));print('wg=$1 xk=$2 xs=$3', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])" || tail -2 gpurun_out/w4c.err
done
