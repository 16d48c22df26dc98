mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests/ > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --routing pinned > gpurun_out/bench_c3_pinned.json 2> gpurun_out/bench_c3_pinned.err
for c in c1 c2; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 16 --out gpurun_out/b200_steps_8b_bf16.json > gpurun_out/grid16.log 2>&1
python scripts/step_timeline.py --config c3 > gpurun_out/tl_c3.txt 2>&1
python scripts/step_timeline.py --config c3 --stamp 4 > gpurun_out/tl_c3_chain.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|gemm_chain|attn_|embed_norm|argmax" -s 68 -c 68 --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_step.py --config c3 --steps 2 > gpurun_out/ncu1_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|gemm_chain|attn_decode" -s 10 -c 5 -o gpurun_out/full_c3 python scripts/profile_step.py --config c3 --steps 1 > gpurun_out/ncu2_c3.log 2>&1
timeout 900 python scripts/scale_emulation.py --config c3 --out gpurun_out/scale_emulation_c3.json > gpurun_out/scale_c3.log 2>&1
