#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py tests/test_checkpoint_gpu.py -k "tiny or serving or bit_identical" > gpurun_out/t_gvc.log 2>&1; tail -2 gpurun_out/t_gvc.log
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "nochain or nogemv or gemv" > gpurun_out/t_gvc2.log 2>&1; tail -2 gpurun_out/t_gvc2.log
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8 --contexts 256,4096 --out gpurun_out/grid_w4_gvc.json 2>&1 | tail -6
python scripts/step_timeline.py --config c4 --batch 1 --isl 256 --layers 2 > gpurun_out/tl_gvc.txt 2>&1; tail -9 gpurun_out/tl_gvc.txt
