mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py tests/test_kernels_gpu.py -k "not subprocess" > gpurun_out/pt_w4j.log 2>&1; echo "rc $?" >> gpurun_out/pt_w4j.log
if grep -q "rc 0" gpurun_out/pt_w4j.log; then
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
P=SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_prev.so
for r in a b; do run c4new$r --config c4; run c4old$r $P --config c4; done
run c3new --config c3; run c3old $P --config c3
timeout 300 python scripts/step_timeline.py --config c4 > gpurun_out/tl_c4_w4j.txt 2>&1
fi
