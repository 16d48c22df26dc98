#!/bin/bash
# QKV -> attention per-tile hand-off (SUN_ATTN_TILE_READY=1): parity, then same-box A/B.
mkdir -p gpurun_out
export SUN_ATTN_TILE_READY=1
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/t_tho.log 2>&1; tail -2 gpurun_out/t_tho.log
timeout 900 python -m pytest -q -x -s -m gpu tests/test_parity_baseline_gpu.py -k "c2 or c3 or c5" > gpurun_out/t_tho_b.log 2>&1; grep -a "c[0-9]:\|passed\|failed" gpurun_out/t_tho_b.log | tail -5
unset SUN_ATTN_TILE_READY
bash scripts/gpu_ab.sh SUN_ATTN_TILE_READY "0 1" c2 c3 c5
