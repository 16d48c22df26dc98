#!/bin/bash
# Same-box A/B of two library builds: scripts/gpu_ab_lib.sh <variant name> cfg1 cfg2 ...
# (default build vs paper_2603_02599_b200/libsun_b200_<variant>.so)
v=$1; shift
L=$PWD/paper_2603_02599_b200
for rep in 1 2; do for cfg in "$@"; do for lib in libsun_b200.so libsun_b200_$v.so; do
  SUN_LIB=$L/$lib timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib', '$cfg', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done; done; done
