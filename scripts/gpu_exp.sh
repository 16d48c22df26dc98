mkdir -p gpurun_out
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run c3s3
run c5s3 --config c5 --steps 20
cp paper_2603_02599_b200/libsun_b200.so /tmp/orig.so
for st in d128s2 d128s4; do cp scripts/exp_libs/lib_$st.so paper_2603_02599_b200/libsun_b200.so; run c3$st; run c5$st --config c5 --steps 20; done
cp /tmp/orig.so paper_2603_02599_b200/libsun_b200.so
