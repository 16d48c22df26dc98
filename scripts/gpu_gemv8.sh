#!/bin/bash
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py tests/test_checkpoint_gpu.py -k "gemv or tiny_variants or bit_identical" > gpurun_out/t_gemv.log 2>&1; tail -2 gpurun_out/t_gemv.log
timeout 120 python scripts/gv_timeline.py 2>&1 | grep -v Warn | cut -c1-240
for cfg in 4:3 2:6 2:4; do kbs=${cfg%%:*}; st=${cfg##*:}; SUN_GV_KBS=$kbs SUN_GV_STAGES=$st TAG=k${kbs}s$st timeout 120 python scripts/gv_timeline.py 2>&1 | grep "B= 1" | cut -c1-200; done
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16 --contexts 256 --out gpurun_out/grid_w4_gemv.json 2>&1 | tail -4
