#!/bin/bash
# Re-measured W4 B=1 timeline (exit stamps after every role) and GEMV vs W4 chain at 9..16 rows.
mkdir -p gpurun_out
python scripts/step_timeline.py --config c4 --batch 1 --isl 256 > gpurun_out/tl_c4_b1.txt 2>&1; tail -7 gpurun_out/tl_c4_b1.txt
timeout 120 python scripts/gv_timeline.py > gpurun_out/gv_timeline.txt 2>&1
for rep in 1 2; do for mb in 8 16; do
  SUN_GV_MAX_BATCH=$mb timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 9,12,16 --contexts 256,2048 --out gpurun_out/grid_mb.json > gpurun_out/grid_mb.log 2>&1
  echo "max_batch=$mb rep=$rep $(grep "ms$" gpurun_out/grid_mb.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
