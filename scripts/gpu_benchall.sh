# All bench configs (N=1) + pinned routing, default flags; lines kept under gpurun_out/bench_*.json
mkdir -p gpurun_out
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --routing pinned > gpurun_out/bench_c3_pinned.json 2> gpurun_out/bench_c3_pinned.err
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
