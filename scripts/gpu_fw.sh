#!/bin/bash
# W4 GEMV first-stage hand-off (SUN_GV_FIRST_WAIT) x ring depth, 8B W4 steps, same box.
for rep in 1 2; do for cfg in "1 2" "0 2" "0 3" "1 3"; do set -- $cfg
  SUN_GV_FIRST_WAIT=$1 SUN_GV_STAGES=$2 timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256,2048 --out gpurun_out/grid_fw.json > gpurun_out/grid_fw.log 2>&1
  echo "first_wait=$1 stages=$2 rep=$rep $(grep "ms$" gpurun_out/grid_fw.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
