#!/bin/bash
# Round-2 re-entry check: GPU suite, smoke, C3 full bench, C2/C4 short benches,
# standalone W4 GEMM probe, C4/C3 step timelines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 600 gpurun_out/bench_c3.json
for cfg in c2 c4; do
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu > gpurun_out/chk_$cfg.json 2> gpurun_out/chk_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/chk_$cfg.json'));print('$cfg', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
PROBE_B=1,4,16,128 timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe.log 2>&1; grep -v "^{" gpurun_out/w4probe.log
timeout 300 python scripts/step_timeline.py --config c4 > gpurun_out/tl_c4.txt 2>&1; tail -30 gpurun_out/tl_c4.txt
timeout 300 python scripts/step_timeline.py --config c3 > gpurun_out/tl_c3.txt 2>&1
