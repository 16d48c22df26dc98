mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/pt_p8.log 2>&1; echo "rc $?" >> gpurun_out/pt_p8.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for r in a b c; do run c3p8$r --config c3; done
run c2p8 --config c2
timeout 300 python scripts/step_timeline.py --config c3 --stamp 4 > gpurun_out/tl_p8_4.txt 2>&1
