#!/bin/bash
# One GPU session: tests, smoke, bench (N=1), launch list + ncu full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|attn_|rmsnorm|argmax" -s 259 -c 259 --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --steps 2 > gpurun_out/ncu1.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attn_decode" -s 12 -c 5 -o gpurun_out/full_c3 python scripts/profile_step.py --steps 1 > gpurun_out/ncu2.log 2>&1
fi
