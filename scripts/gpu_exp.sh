mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 20 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run c5 --config c5
run c5fc SUN_ATTN_FUSED_COMBINE=1 --config c5
for p in 64 128 256; do run c5p$p --config c5 --pps $p; done
