mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run c3
run c4 --config c4 --steps 20
for k in 1 16; do run skip$k SUN_SKIP_KERNELS=$k; done
