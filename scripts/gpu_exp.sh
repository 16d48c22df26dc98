mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py -x -k "attention or tiny" > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for p in 0 20 32 44 100; do run pps$p --pps $p; done
for p in 0 64 128 300; do run c4pps$p --pps $p --config c4 --steps 20; done
