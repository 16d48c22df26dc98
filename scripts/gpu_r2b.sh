#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --config c5 --steps 30 --warmup 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 400 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 1500 python -m pytest -q -s -m gpu tests/test_parity_baseline_gpu.py > gpurun_out/parity_baseline.log 2>&1; tail -12 gpurun_out/parity_baseline.log
