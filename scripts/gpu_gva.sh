#!/bin/bash
# W4 GEMV with a dedicated epilogue group (SUN_GV_ASYNC_EPI) x balanced schedule (SUN_GV_BALANCE):
# tests, per-CTA stamps, same-box 8B W4 steps.
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "gemv or gvbal" > gpurun_out/t_gva.log 2>&1; tail -2 gpurun_out/t_gva.log
timeout 600 python -m pytest -q -x -s -m gpu tests/test_parity_baseline_gpu.py -k c4s > gpurun_out/t_c4s.log 2>&1; grep -a "c4s:\|passed\|failed" gpurun_out/t_c4s.log | tail -3
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
  echo "== SUN_GV_ASYNC_EPI=$1 SUN_GV_BALANCE=$2"; SUN_GV_ASYNC_EPI=$1 SUN_GV_BALANCE=$2 timeout 120 python scripts/gv_timeline.py 2>&1 | grep -v Warn | cut -c1-200
done
for rep in 1 2; do for cfg in "0 0" "1 0" "1 1" "1 2"; do set -- $cfg
  SUN_GV_ASYNC_EPI=$1 SUN_GV_BALANCE=$2 timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256,2048 --out gpurun_out/grid_gva.json > gpurun_out/grid_gva.log 2>&1
  echo "async=$1 bal=$2 rep=$rep $(grep "ms$" gpurun_out/grid_gva.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
