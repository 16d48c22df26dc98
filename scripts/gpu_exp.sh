mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for r in a b; do for o in 0 2 4 6; do run c3p$o$r SUN_CHAIN_OPTS=$o --config c3; done; done
for o in 0 6; do run c2p$o SUN_CHAIN_OPTS=$o --config c2; done
