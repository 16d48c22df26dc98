#!/bin/bash
# Small-batch W4 GEMV: its GPU tests, per-CTA phase stamps of the standalone kernel
# (scripts/gv_timeline.py) and 8B W4 decode steps at B <= 16.
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py tests/test_checkpoint_gpu.py -k "gemv or tiny_variants or bit_identical" > gpurun_out/t_gemv.log 2>&1; tail -2 gpurun_out/t_gemv.log
timeout 120 python scripts/gv_timeline.py 2>&1 | grep -v Warn | cut -c1-240
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16 --contexts 256 --out gpurun_out/grid_w4_gemv.json 2>&1 | tail -4
