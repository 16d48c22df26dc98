mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python scripts/prefill_speed.py > gpurun_out/prefill.txt 2>&1
