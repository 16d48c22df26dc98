mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py tests/test_serving_gpu.py -k "not subprocess" > gpurun_out/pt_pre.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_pre.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for c in c3 c2 c4 c5; do
run ${c}pre1 --config $c
run ${c}pre0 SUN_ATTN_PRESTAGE=0 --config $c
done
run c3pre1b --config c3
run c3pre0b SUN_ATTN_PRESTAGE=0 --config c3
run c3chain SUN_GEMM_CHAIN=1 --config c3
timeout 300 python scripts/step_timeline.py --config c3 > gpurun_out/tl_pre.txt 2>&1
