#!/bin/bash
L=$PWD/paper_2603_02599_b200
SUN_LIB=$L/libsun_b200_gvidle.so TAG=idle timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"
for st in 4 5 6; do SUN_LIB=$L/libsun_b200_gvidlenox.so SUN_GV_STAGES=$st TAG=idlenox_st$st timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"; done
for st in 5 6; do SUN_LIB=$L/libsun_b200_gvnox.so SUN_GV_STAGES=$st TAG=nox_st$st timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1"; done
