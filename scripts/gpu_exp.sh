mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/pt_l1.log 2>&1; echo "rc $?" >> gpurun_out/pt_l1.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for r in a b; do for o in 1 0; do run c3l1$o$r SUN_CHAIN_L1PF=$o --config c3; done; done
for o in 1 0; do run c2l1$o SUN_CHAIN_L1PF=$o --config c2; run c5l1$o SUN_CHAIN_L1PF=$o --config c5; done
