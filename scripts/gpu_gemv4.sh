#!/bin/bash
mkdir -p gpurun_out
L=$PWD/paper_2603_02599_b200
timeout 120 python scripts/gv_timeline.py 2>&1 | grep -v Warn
for v in gvnomma gvnocvt; do SUN_LIB=$L/libsun_b200_$v.so timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"; done
SUN_GV_KBS=2 TAG=kbs2 timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"
SUN_GV_KBS=1 TAG=kbs1 timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"
SUN_GV_KBS=2 SUN_GV_CTAS_PER_SM=2 TAG=kbs2x2 timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"
