mkdir -p gpurun_out
timeout 900 python scripts/scale_emulation.py --config c3 --out gpurun_out/scale_emulation_c3.json > gpurun_out/scale_c3.log 2>&1
timeout 900 python scripts/scale_emulation.py --config c5 --cap 40 --reps 10 --out gpurun_out/scale_emulation_c5.json > gpurun_out/scale_c5.log 2>&1
timeout 300 python scripts/step_timeline.py --config c3 --stamp 4 > gpurun_out/tl_c3_chain.txt 2>&1
