#!/bin/bash
# W4 small-batch evidence: ncu launch list of one B=1 decode step (GEMV launches), a full
# capture of the gate_up GEMV (standalone, B=1), per-CTA stamps of the GEMV shapes.
mkdir -p gpurun_out
python scripts/step_timeline.py --config c4 --batch 1 --isl 256 > gpurun_out/tl_c4_b1.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv_w4|gemm_kernel|attn_|embed_norm|argmax" -s 195 -c 195 --csv --log-file gpurun_out/launches_w4_b1.csv python scripts/profile_step.py --config c4 --batch 1 --isl 256 --steps 2 > gpurun_out/ncu_w4b1.log 2>&1; tail -2 gpurun_out/ncu_w4b1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_w4 -s 1 -c 1 -o gpurun_out/gv_full_b1 python scripts/gv_one.py > gpurun_out/ncu_gv.log 2>&1; tail -1 gpurun_out/ncu_gv.log
timeout 120 python scripts/gv_timeline.py > gpurun_out/gv_timeline.txt 2>&1
