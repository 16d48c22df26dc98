mkdir -p gpurun_out
export SUN_GEMM_CHAIN=1
timeout 300 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py -x > gpurun_out/pytest_chain.log 2>&1; tail -1 gpurun_out/pytest_chain.log
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/x_chain.json 2>gpurun_out/x_chain.err
timeout 300 python bench.py --config c2 --steps 30 --no-cpu --no-e2e > gpurun_out/x_chain_c2.json 2>gpurun_out/x_chain_c2.err
timeout 300 python bench.py --config c5 --steps 20 --no-cpu --no-e2e > gpurun_out/x_chain_c5.json 2>gpurun_out/x_chain_c5.err
unset SUN_GEMM_CHAIN
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/x_base.json 2>gpurun_out/x_base.err
