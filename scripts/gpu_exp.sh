mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for kb in 0 64 128 256 512; do run pf$kb SUN_GEMM_PREFETCH_KB=$kb; done
for kb in 0 128 512; do run c4pf$kb SUN_GEMM_PREFETCH_KB=$kb --config c4 --steps 20; done
