#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py -k "gemv or tiny_variants" > gpurun_out/t_gemv.log 2>&1; tail -2 gpurun_out/t_gemv.log
PROBE_GEMV=1 PROBE_B=1,16 timeout 300 python scripts/w4_probe.py > gpurun_out/gvprobe.log 2>&1; grep W4 gpurun_out/gvprobe.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_w4 -s 1 -c 1 -o gpurun_out/gv_full_b1 python scripts/gv_one.py > gpurun_out/ncu_gv.log 2>&1; tail -1 gpurun_out/ncu_gv.log
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16 --contexts 256 --out gpurun_out/grid_w4_gemv.json 2>&1 | tail -4
