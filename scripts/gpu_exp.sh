mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/pt_noinl.log 2>&1; echo "rc $?" >> gpurun_out/pt_noinl.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
P=SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_prev.so
for r in a b c; do run c3ni$r --config c3; run c3oi$r $P --config c3; done
run c2ni --config c2; run c2oi $P --config c2
