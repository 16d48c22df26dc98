#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py -k "qsun or tiny" > gpurun_out/w4c_parity_tiny.log 2>&1; tail -1 gpurun_out/w4c_parity_tiny.log
timeout 600 python -m pytest -q -x -s -m gpu tests/test_parity_baseline_gpu.py -k c4 > gpurun_out/w4c_parity_c4.log 2>&1; grep -E "c4:|passed|failed" gpurun_out/w4c_parity_c4.log | tail -2
timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/w4c_bench_c4.json 2> gpurun_out/w4c_bench_c4.err; python -c "import json;d=json.load(open('gpurun_out/w4c_bench_c4.json'));print('chain c4', d['ms_per_step'], d.get('kernel_ms_per_step'))"
timeout 200 python scripts/step_timeline.py --config c4 --stamp 4 > gpurun_out/tl_c4_chain.txt 2>&1; tail -17 gpurun_out/tl_c4_chain.txt
timeout 400 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,16,64,128 --contexts 256,4096 --reps 10 --out gpurun_out/w4c_grid.json > gpurun_out/w4c_grid.log 2>&1; tail -8 gpurun_out/w4c_grid.log
