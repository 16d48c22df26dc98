mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ -x -k "w4 or W4 or variants or tiny" > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python scripts/w4_sweep.py > gpurun_out/w4_sweep.txt 2>&1
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run c4 --config c4 --steps 20
run c4x3 SUN_W4_XSTAGES=3 --config c4 --steps 20
