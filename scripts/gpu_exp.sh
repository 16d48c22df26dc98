mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pt_chain.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_chain.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 300 python scripts/step_timeline.py --config c3 > gpurun_out/tl_chain.txt 2>&1
timeout 300 python bench.py --steps 50 > gpurun_out/x_c3full.json 2>gpurun_out/x_c3full.err
