mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --config c2 --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c1 --steps 30 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
