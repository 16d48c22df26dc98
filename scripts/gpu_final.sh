#!/bin/bash
# Round-end state check: full GPU suite, smoke, the default bench line (C3, N=1), reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu_final.log 2>&1; tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -1 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default.err
