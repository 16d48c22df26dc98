mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_decode_parity_gpu.py tests/test_serving_gpu.py -x > gpurun_out/pytest_flow.log 2>&1; tail -1 gpurun_out/pytest_flow.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run flow
run noflow SUN_GEMM_FLOW=0
run flowvcl SUN_GEMM_VCLUSTER=2
run c2flow --config c2 --steps 30
run c5flow --config c5 --steps 20
python scripts/step_timeline.py --config c3 > gpurun_out/tl_flow.txt 2>&1
