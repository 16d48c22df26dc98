mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py -x > gpurun_out/pytest_grp.log 2>&1; tail -3 gpurun_out/pytest_grp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python scripts/prefill_speed.py > gpurun_out/prefill.txt 2>&1
