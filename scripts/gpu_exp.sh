mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run c3
run c4 --config c4 --steps 20
python scripts/step_timeline.py --config c3 > gpurun_out/tl_c3.txt 2>&1
