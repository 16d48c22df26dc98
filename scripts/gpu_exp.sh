mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c2 --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python scripts/scale_emulation.py --config c3 --out gpurun_out/scale_emulation_c3.json > gpurun_out/scale_c3.log 2>&1
timeout 900 python scripts/scale_emulation.py --config c5 --cap 40 --reps 10 --out gpurun_out/scale_emulation_c5.json > gpurun_out/scale_c5.log 2>&1
