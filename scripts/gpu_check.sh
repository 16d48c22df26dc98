#!/bin/bash
# Quick check: GPU suite, smoke, 8B W4 step grid at ctx 256, a short C4 bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,4,8,16,64,128 --contexts 256 --out gpurun_out/grid_w4.json 2>&1 | tail -6
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/chk_c4.json 2> gpurun_out/chk_c4.err
python -c "import json;d=json.load(open('gpurun_out/chk_c4.json'));print('c4', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s', d['roofline']['kernel'], round(d['roofline']['frac'],3))"
for c in c2 c3; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-handoff > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err
  python -c "import json;d=json.load(open('gpurun_out/chk_$c.json'));print('$c', round(d['ms_per_step'],4), 'ms', round(d['value']), 'tok/s', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/chk_$c.err
done
