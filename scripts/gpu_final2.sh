#!/bin/bash
# Final tree: full GPU suite, smoke, default bench, W4 small-batch grid, W4 B=1 step timeline + launch list.
bash scripts/gpu_final.sh
timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8 --contexts 256,1024,2048,4096 --out gpurun_out/grid_w4_small.json 2>&1 | grep "ms$"
python scripts/step_timeline.py --config c4 --batch 1 --isl 256 > gpurun_out/tl_c4_b1.txt 2>&1; tail -7 gpurun_out/tl_c4_b1.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv_w4|gemm_kernel|attn_|embed_norm|argmax" -s 195 -c 195 --csv --log-file gpurun_out/launches_w4_b1.csv python scripts/profile_step.py --config c4 --batch 1 --isl 256 --steps 2 > gpurun_out/ncu_w4b1.log 2>&1; tail -1 gpurun_out/ncu_w4b1.log
timeout 120 python scripts/gv_timeline.py > gpurun_out/gv_timeline.txt 2>&1
