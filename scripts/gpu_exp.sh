mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
P=SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200_prev.so
for r in a b; do run c3new$r --config c3; run c3old$r $P --config c3; done
run c5new --config c5; run c5old $P --config c5
run c2new --config c2; run c2old $P --config c2
