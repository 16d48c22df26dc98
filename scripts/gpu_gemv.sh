#!/bin/bash
# Small-batch W4 GEMV bring-up: its tests, standalone timings vs the tcgen05 W4 GEMM,
# and 8B W4 decode steps at B <= 16 with and without it.
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py -k "gemv" > gpurun_out/t_gemv.log 2>&1; tail -3 gpurun_out/t_gemv.log
timeout 900 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py tests/test_checkpoint_gpu.py -k "tiny_variants or checkpoint or import or bit_identical" > gpurun_out/t_gemv2.log 2>&1; tail -3 gpurun_out/t_gemv2.log
PROBE_B=1,4,9,16 timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe_tc.log 2>&1
PROBE_GEMV=1 PROBE_B=1,4,9,16 timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe_gemv.log 2>&1
paste <(grep W4 gpurun_out/w4probe_tc.log) <(grep W4 gpurun_out/w4probe_gemv.log | awk '{print $(NF-3), $(NF-2), $(NF-1), $NF}')
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16 --contexts 256 --out gpurun_out/grid_w4_gemv.json 2>&1 | tail -4
SUN_W4_GEMV=0 timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16 --contexts 256 --out gpurun_out/grid_w4_tc.json 2>&1 | tail -4
