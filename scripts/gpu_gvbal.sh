#!/bin/bash
# W4 GEMV balanced schedule (SUN_GV_BALANCE 0 / 1 / 2): tests, per-CTA stamps, same-box 8B W4 steps.
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "gemv or gvbal" > gpurun_out/t_gvbal.log 2>&1; tail -2 gpurun_out/t_gvbal.log
timeout 600 python -m pytest -q -x -s -m gpu tests/test_parity_baseline_gpu.py -k c4s > gpurun_out/t_c4s.log 2>&1; grep -a "c4s:\|passed\|failed" gpurun_out/t_c4s.log | tail -3
for b in 0 1 2; do
  echo "== SUN_GV_BALANCE=$b"; SUN_GV_BALANCE=$b timeout 120 python scripts/gv_timeline.py 2>&1 | grep -v Warn | cut -c1-200
done
for rep in 1 2; do for b in 0 1 2; do
  SUN_GV_BALANCE=$b timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256 --out gpurun_out/grid_gvbal$b.json > gpurun_out/grid_gvbal$b.log 2>&1
  echo "bal=$b rep=$rep $(grep "ms$" gpurun_out/grid_gvbal$b.log | tr "\n" " ")"
done; done
