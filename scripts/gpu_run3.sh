mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/ -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for sch in 0 1; do SUN_GEMM_SCHED=$sch timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > gpurun_out/b3_s$sch.json 2>gpurun_out/b3_s$sch.err; done
for sch in 0 1; do SUN_GEMM_SCHED=$sch timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > gpurun_out/b4_s$sch.json 2>gpurun_out/b4_s$sch.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 2 -c 4 -o gpurun_out/full_c4 python scripts/profile_step.py --config c4 --steps 1 > gpurun_out/ncu_c4.log 2>&1
