#!/bin/bash
# One GPU session: tests, smoke, bench (N=1), launch list + ncu full captures (C3, C4).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ "$1" == "ncu" ]; then
  for cfg in c3 c4; do
    # one decode step = 163 launches (embed + 32 x 5 + lm_head + argmax; unsplit attention, no combine): skip the first step, capture the second
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|attn_|embed_norm|argmax" -s 163 -c 163 --csv --log-file gpurun_out/launches_$cfg.csv python scripts/profile_step.py --config $cfg --steps 2 > gpurun_out/ncu1_$cfg.log 2>&1
    # one layer (layer 2): QKV, attention, O, gate_up, down
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|attn_decode" -s 10 -c 5 -o gpurun_out/full_$cfg python scripts/profile_step.py --config $cfg --steps 1 > gpurun_out/ncu2_$cfg.log 2>&1
  done
fi
