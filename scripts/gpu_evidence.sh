#!/bin/bash
# Round-2 evidence: GPU tests, smoke, every bench config (N=1) + pinned + reference arm,
# step-time grids (harness closure fixtures), step timelines, ncu launch lists + full
# captures (C3, C4) -> gpurun_out/ (copied to profiles/<round> by hand).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --routing pinned > gpurun_out/bench_c3_pinned.json 2> gpurun_out/bench_c3_pinned.err
for c in c1 c2 c4 c5; do timeout 1500 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 16 --out gpurun_out/b200_steps_8b_bf16.json > gpurun_out/grid16.log 2>&1
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --out gpurun_out/b200_steps_8b_w4.json > gpurun_out/grid4.log 2>&1
for cfg in c3 c4 c2; do python scripts/step_timeline.py --config $cfg > gpurun_out/tl_$cfg.txt 2>&1; done
python scripts/step_timeline.py --config c4 --batch 1 --isl 256 > gpurun_out/tl_c4_b1.txt 2>&1
for cl in c3:68 c4:68; do
  cfg=${cl%%:*}; nl=${cl##*:}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|gemm_chain|gemv_w4|attn_|embed_norm|argmax" -s $nl -c $nl --csv --log-file gpurun_out/launches_$cfg.csv python scripts/profile_step.py --config $cfg --steps 2 > gpurun_out/ncu1_$cfg.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_chain|attn_decode" -s 4 -c 2 -o gpurun_out/full_$cfg python scripts/profile_step.py --config $cfg --steps 1 > gpurun_out/ncu2_$cfg.log 2>&1
done
# small-batch QSUN (8B W4, B=1, ctx 256): one step's launch list, per-CTA GEMV stamps
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|gemm_chain|gemv_w4|attn_|embed_norm|argmax" -s 195 -c 195 --csv --log-file gpurun_out/launches_w4_b1.csv python scripts/profile_step.py --config c4 --batch 1 --isl 256 --steps 2 > gpurun_out/ncu1_w4_b1.log 2>&1
timeout 300 python scripts/gv_timeline.py > gpurun_out/gemv_w4_cta_stamps.txt 2>&1
# per-CTA phase stamps of one layer chain (C2 bf16, C4 W4)
python scripts/step_timeline.py --config c2 --layers 1 --stamp 4 > gpurun_out/tl_c2_chain.txt 2>&1
python scripts/step_timeline.py --config c4 --layers 1 --stamp 4 > gpurun_out/tl_c4_chain.txt 2>&1
# BASELINE-shape parity log
timeout 1200 python -m pytest -q -s -m gpu tests/test_parity_baseline_gpu.py > gpurun_out/parity_baseline.log 2>&1; tail -1 gpurun_out/parity_baseline.log
