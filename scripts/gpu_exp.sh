mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for c in c5 c3 c2 c1; do for o in 1 0; do run ${c}hv$o SUN_CHAIN_CLUSTER=$o --config $c; done; done
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pt_hv.log 2>&1; echo "rc $?" >> gpurun_out/pt_hv.log
