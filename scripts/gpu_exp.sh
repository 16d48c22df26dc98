mkdir -p gpurun_out
SUN_CHAIN_VCL8=1 timeout 600 python -m pytest -q -x -m gpu tests/test_decode_parity_gpu.py > gpurun_out/pt_v8.log 2>&1; echo "rc $?" >> gpurun_out/pt_v8.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
for r in a b; do run c2v1$r SUN_CHAIN_VCL8=1 --config c2; run c2v0$r --config c2; done
run c1v1 SUN_CHAIN_VCL8=1 --config c1; run c1v0 --config c1
