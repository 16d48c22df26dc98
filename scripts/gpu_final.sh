#!/bin/bash
# End-of-round evidence: GPU tests, smoke, every bench config (N=1) + pinned + reference
# arm, step-time grids (harness closure fixtures), ncu launch lists + full captures (C3, C4).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --routing pinned > gpurun_out/bench_c3_pinned.json 2> gpurun_out/bench_c3_pinned.err
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 16 --out gpurun_out/b200_steps_8b_bf16.json > gpurun_out/grid16.log 2>&1
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --out gpurun_out/b200_steps_8b_w4.json > gpurun_out/grid4.log 2>&1
# launches per step: C3 (bf16 layer chain) embed + qkv + 32 x (attention, chain) + lm_head + argmax = 68;
# C4 (QSUN, separate GEMMs, unsplit attention) 1 + 32 x 5 + 2 = 163
for cl in c3:68 c4:163; do
  cfg=${cl%%:*}; nl=${cl##*:}
  python scripts/step_timeline.py --config $cfg > gpurun_out/tl_$cfg.txt 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|gemm_chain|attn_|embed_norm|argmax" -s $nl -c $nl --csv --log-file gpurun_out/launches_$cfg.csv python scripts/profile_step.py --config $cfg --steps 2 > gpurun_out/ncu1_$cfg.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|gemm_chain|attn_decode" -s 10 -c 5 -o gpurun_out/full_$cfg python scripts/profile_step.py --config $cfg --steps 1 > gpurun_out/ncu2_$cfg.log 2>&1
done
