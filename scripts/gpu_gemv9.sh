#!/bin/bash
L=$PWD/paper_2603_02599_b200
for v in gvidle gvnox gvnocvt; do SUN_LIB=$L/libsun_b200_$v.so TAG=$v timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1" | cut -c1-250; done
