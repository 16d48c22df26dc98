mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run base SUN_GEMM_SCHED=0
run sk SUN_GEMM_SCHED=1
run sk4 SUN_GEMM_SCHED=1 --config c4
run base4 SUN_GEMM_SCHED=0 --config c4
SLOW=1 SUN_GEMM_SCHED=1 python scripts/gemm_timeline.py > gpurun_out/timeline_sk.txt 2>&1
