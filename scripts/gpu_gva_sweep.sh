#!/bin/bash
# W4 GEMV (dedicated epilogue group) ring depth sweep: 8B W4 steps at B=1 / 8, ctx 256, same box.
for rep in 1 2; do for st in 2 3 4; do
  SUN_GV_STAGES=$st timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256 --out gpurun_out/grid_sw.json > gpurun_out/grid_sw.log 2>&1
  echo "stages=$st rep=$rep $(grep "ms$" gpurun_out/grid_sw.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
