#!/bin/bash
# Epilogue-group GEMV: four partials per L2 round trip at NB = 1 (tests, then same-box A/B vs the previous build)
timeout 600 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "gemv and not subprocess" 2>&1 | tail -1 | sed "s/^/gemv tests: /"
timeout 300 python -m pytest -q -s -m gpu tests/test_parity_baseline_gpu.py -k c4s 2>&1 | grep -a "c4s:\|passed\|failed" | tail -2
for rep in 1 2; do for lib in default prev; do
  if [ $lib = default ]; then unset SUN_LIB; else export SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_$lib.so; fi
  timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,8 --contexts 256,2048 --out gpurun_out/grid_pf.json > gpurun_out/grid_pf.log 2>&1
  echo "$lib rep=$rep $(grep "ms$" gpurun_out/grid_pf.log | sed 's/ctx=//;s/B=//' | tr -s ' ' | tr "\n" ";")"
done; done
unset SUN_LIB
