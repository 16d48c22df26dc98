mkdir -p gpurun_out
timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py -s > gpurun_out/pt_fs.log 2>&1; echo "rc $?" >> gpurun_out/pt_fs.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for c in c3 c2 c3 c2; do run ${c}fs --config $c; done
timeout 300 python scripts/step_timeline.py --config c3 --stamp 4 > gpurun_out/tl_fs_4.txt 2>&1
