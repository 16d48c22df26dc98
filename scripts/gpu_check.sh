#!/bin/bash
# Full GPU suite + smoke + short C3/C4 benches
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for cfg in c3 c4; do
  timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu > gpurun_out/chk_$cfg.json 2> gpurun_out/chk_$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/chk_$cfg.json'));print('$cfg', round(d['ms_per_step'],3), 'ms', round(d['value']), 'tok/s e2e', round(d['e2e']['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
