mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --config c4 --steps 30 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --out gpurun_out/b200_steps_8b_w4.json > gpurun_out/grid4.log 2>&1
python scripts/step_timeline.py --config c4 > gpurun_out/tl_c4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|gemm_chain|attn_|embed_norm|argmax" -s 163 -c 163 --csv --log-file gpurun_out/launches_c4.csv python scripts/profile_step.py --config c4 --steps 2 > gpurun_out/ncu1_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|gemm_chain|attn_decode" -s 10 -c 5 -o gpurun_out/full_c4 python scripts/profile_step.py --config c4 --steps 1 > gpurun_out/ncu2_c4.log 2>&1
