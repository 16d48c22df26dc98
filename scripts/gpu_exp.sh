mkdir -p gpurun_out
for cfg in c3 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|attn_|embed_norm|argmax" -s 163 -c 163 --csv --log-file gpurun_out/launches_$cfg.csv python scripts/profile_step.py --config $cfg --steps 2 > gpurun_out/ncu1_$cfg.log 2>&1
done
timeout 1500 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
SUN_GEMM_VCL_OWNER=1 timeout 1500 python -m pytest -q -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py -x > gpurun_out/pytest_owner.log 2>&1; tail -1 gpurun_out/pytest_owner.log
SUN_GEMM_VCL_OWNER=1 SUN_GEMM_VCLUSTER=2 timeout 1500 python -m pytest -q -m gpu tests/test_kernels_gpu.py tests/test_decode_parity_gpu.py -x > gpurun_out/pytest_owner2.log 2>&1; tail -1 gpurun_out/pytest_owner2.log
run() { tag=$1; shift; e=(); while [[ "$1" == *=* ]]; do e+=("$1"); shift; done; env "${e[@]}" timeout 300 python bench.py --steps 50 --no-cpu --no-e2e "$@" > gpurun_out/x_$tag.json 2>gpurun_out/x_$tag.err; }
run base
run own SUN_GEMM_VCL_OWNER=1
run own2 SUN_GEMM_VCL_OWNER=1 SUN_GEMM_VCLUSTER=2
run vcl2 SUN_GEMM_VCLUSTER=2
run c4own SUN_GEMM_VCL_OWNER=1 --config c4 --steps 20
run c2own2 SUN_GEMM_VCL_OWNER=1 SUN_GEMM_VCLUSTER=2 --config c2 --steps 30
run c2base --config c2 --steps 30
SUN_GEMM_VCL_OWNER=1 SUN_GEMM_VCLUSTER=2 python scripts/step_timeline.py --config c3 > gpurun_out/tl_own2.txt 2>&1
