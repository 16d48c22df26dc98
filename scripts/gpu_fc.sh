#!/bin/bash
# Same-box A/B: fused split-combine in the attention kernel (SUN_ATTN_FUSED_COMBINE) at small batches.
mkdir -p gpurun_out
for rep in 1 2; do for bits in 4 16; do for v in 0 1; do
  SUN_ATTN_FUSED_COMBINE=$v timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits $bits --batches 1,8,32 --contexts 256,2048 --out gpurun_out/grid_fc.json > gpurun_out/grid_fc.log 2>&1
  echo "fc=$v bits=$bits rep=$rep $(grep "ms$" gpurun_out/grid_fc.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done; done
