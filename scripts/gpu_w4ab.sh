#!/bin/bash
# Same-box A/B of QSUN chain variants: C4 bench + small-batch W4 step grid, per (library, env) combination
mkdir -p gpurun_out; : > gpurun_out/w4ab.log
for lib in "" _nogb; do
  for cl in 1 0; do
    for chain in 1 0; do
      [ "$chain" == 0 ] && [ "$cl" == 0 ] && continue
      [ "$chain" == 0 ] && [ "$lib" == "_nogb" ] && continue
      tag="lib=${lib:-default} cluster=$cl chain=$chain"
      export SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200$lib.so SUN_CHAIN_CLUSTER=$cl
      if [ "$chain" == 0 ]; then export SUN_GEMM_CHAIN=0; else unset SUN_GEMM_CHAIN; fi
      timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu --no-e2e > /tmp/b.json 2>/dev/null
      c4=$(python -c "import json;print(round(json.load(open('/tmp/b.json'))['ms_per_step'],3))" 2>/dev/null)
      timeout 300 python scripts/measure_step_grid.py --spec llama3.1-8b --bits 4 --batches 1,16,64 --contexts 256 --reps 10 --out /tmp/g.json > /tmp/g.log 2>&1
      echo "$tag | c4 $c4 ms | $(grep 'B=' /tmp/g.log | tr '\n' ' ')" >> gpurun_out/w4ab.log
    done
  done
done
cat gpurun_out/w4ab.log
