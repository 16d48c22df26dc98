mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/w4_sweep.py > gpurun_out/w4_sweep.txt 2>&1
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > gpurun_out/x_c4.json 2>gpurun_out/x_c4.err
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/x_c3.json 2>gpurun_out/x_c3.err
