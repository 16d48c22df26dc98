mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/pt_hw2.log 2>&1; echo "rc $?" >> gpurun_out/pt_hw2.log
if grep -q "rc 0" gpurun_out/pt_hw2.log; then
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for r in a b; do for o in 1 0; do run c3h2$o$r SUN_CHAIN_HW2=$o --config c3; done; done
for o in 1 0; do run c2h2$o SUN_CHAIN_HW2=$o --config c2; done
timeout 300 python scripts/step_timeline.py --config c3 --stamp 4 > gpurun_out/tl_hw2_4.txt 2>&1
fi
