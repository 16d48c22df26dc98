#!/bin/bash
# W4 GEMV defaults check: GEMV tests + schedule subprocesses, c4s parity, evidence, step grid.
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "gemv or gv" > gpurun_out/t_gva.log 2>&1; tail -2 gpurun_out/t_gva.log
timeout 600 python -m pytest -q -x -s -m gpu tests/test_parity_baseline_gpu.py -k c4s > gpurun_out/t_c4s.log 2>&1; grep -a "c4s:\|passed\|failed" gpurun_out/t_c4s.log | tail -3
bash scripts/gpu_gv_evidence.sh
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8 --contexts 256,1024,2048,4096 --out gpurun_out/grid_w4_small.json 2>&1 | grep "ms$"
