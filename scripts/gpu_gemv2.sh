#!/bin/bash
mkdir -p gpurun_out
for v in "" _gvnomma _gvnocvt; do
  SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200$v.so PROBE_GEMV=1 PROBE_B=1,16 timeout 300 python scripts/w4_probe.py > gpurun_out/gvprobe$v.log 2>&1
  grep W4 gpurun_out/gvprobe$v.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_w4 -s 1 -c 1 -o gpurun_out/gv_full_b1 python scripts/gv_one.py > gpurun_out/ncu_gv.log 2>&1; tail -2 gpurun_out/ncu_gv.log
