mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
P=SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_prev.so
for r in a b; do run c5w16$r --config c5; run c5w8$r $P --config c5; done
run c1w16 --config c1; run c1w8 $P --config c1
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py > gpurun_out/pt_w16.log 2>&1; echo "rc $?" >> gpurun_out/pt_w16.log
