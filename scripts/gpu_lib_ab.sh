#!/bin/bash
# Same-box A/B of two library builds: scripts/gpu_lib_ab.sh <variant-name> cfg1 cfg2 ...
# (the in-tree default build vs paper_2603_02599_b200/libsun_b200_<variant-name>.so)
v=$1; shift
for rep in 1 2; do for cfg in "$@"; do for lib in default $v; do
  if [ $lib = default ]; then unset SUN_LIB; else export SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_$lib.so; fi
  timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$lib', '$cfg', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.err
done; done; done
unset SUN_LIB
