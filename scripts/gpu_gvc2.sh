#!/bin/bash
for pre in 0 1 2 4; do
  echo "SUN_GVC_PRE=$pre"; SUN_GVC_PRE=$pre timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256 --reps 10 --out /tmp/g.json 2>&1 | tail -2
done
SUN_GEMM_CHAIN=0 timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256 --reps 10 --out /tmp/g.json 2>&1 | tail -2
SUN_GVC_PRE=1 python scripts/step_timeline.py --config c4 --batch 1 --isl 256 --layers 1 --stamp 4 2>&1 | tail -16
