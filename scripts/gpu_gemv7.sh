#!/bin/bash
L=$PWD/paper_2603_02599_b200
for cfg in 4:4 4:3 4:2 2:6 2:4 2:3 1:8 1:6; do
  kbs=${cfg%%:*}; st=${cfg##*:}
  SUN_LIB=$L/libsun_b200_gvidle.so SUN_GV_KBS=$kbs SUN_GV_STAGES=$st TAG=idle_k${kbs}s$st timeout 120 python scripts/gv_timeline.py 2>&1 | grep "28672x4096 B= 1" | cut -c1-200
  SUN_GV_KBS=$kbs SUN_GV_STAGES=$st TAG=full_k${kbs}s$st timeout 120 python scripts/gv_timeline.py 2>&1 | grep "28672x4096 B= 1" | cut -c1-200
done
