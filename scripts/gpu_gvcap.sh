#!/bin/bash
# W4 GEMV split cap (SUN_GV_SPLIT_CAP) x first-stage hand-off: 8B W4 steps at B=1 / 8, same box.
for rep in 1 2; do for cap in 0 2 3; do
  SUN_GV_SPLIT_CAP=$cap timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256,2048 --out gpurun_out/grid_cap.json > gpurun_out/grid_cap.log 2>&1
  echo "cap=$cap rep=$rep $(grep "ms$" gpurun_out/grid_cap.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
