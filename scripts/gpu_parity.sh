#!/bin/bash
# GPU session: BASELINE-shape parity + long-context attention + W4 GEMM timeline
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest -q -s -m gpu tests/test_parity_baseline_gpu.py > gpurun_out/parity_baseline.log 2>&1; tail -5 gpurun_out/parity_baseline.log
timeout 600 python -m pytest -q -m gpu tests/test_kernels_gpu.py -k "long_context" > gpurun_out/attn_long.log 2>&1; tail -3 gpurun_out/attn_long.log
timeout 300 python scripts/w4_timeline.py > gpurun_out/w4_timeline.log 2>&1; tail -30 gpurun_out/w4_timeline.log
