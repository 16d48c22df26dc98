mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py -k "bit_exact" > gpurun_out/pt_host.log 2>&1; echo "rc $?" >> gpurun_out/pt_host.log
for r in a b; do timeout 300 python bench.py --steps 50 --no-cpu > gpurun_out/x_e2e$r.json 2>gpurun_out/x_e2e$r.err; done
