"""Measure B200 decode-step times over a (batch, context) grid for one decoder
shape, for the harness closure (pricing.fit_decode_step / MeasuredBackend):
each point is a CUDA-graph step over a seeded paged pool, timed with CUDA events
(median of `--reps` steps after warm-up). Output: JSON list of points.

  python scripts/measure_step_grid.py --spec llama3.1-8b --bits 16 --out tests/golden/b200_steps_8b.json
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_02599_b200.kvpool import KvPool, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

ap = argparse.ArgumentParser()
ap.add_argument("--spec", default="llama3.1-8b")
ap.add_argument("--bits", type=int, default=16)
ap.add_argument("--batches", default="1,8,16,32,64,128")
ap.add_argument("--contexts", default="256,1024,2048,4096")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--pps", type=int, default=0, help="attention pages per split (0 = automatic)")
ap.add_argument("--out", required=True)
args = ap.parse_args()

spec = SPECS[args.spec].with_bits(4) if args.bits == 4 else SPECS[args.spec]
dev = torch.device("cuda")
batches = [int(x) for x in args.batches.split(",")]
contexts = [int(x) for x in args.contexts.split(",")]
B_max, C_max = max(batches), max(contexts) + args.reps + 64
dw = DeviceWeights(spec, init_weights(spec, 0, dev), dev, C_max, free_source=True)
kv = KvPool(spec, B_max * pages_for(C_max) + 4, dev)
kv.fill_random_(1)
dec = SharedDecodeModule(spec, dw, kv, B_max, C_max)
for i in range(B_max):
    n = pages_for(C_max)
    dec.block_tables[i, :n] = torch.arange(i * n, (i + 1) * n, dtype=torch.int32, device=dev)
points = []
for ctx in contexts:
    for B in batches:
        dec.positions[:B] = ctx
        for _ in range(3):
            dec.step_static(B, args.pps, graph=True, feedback=False)
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec.step_static(B, args.pps, graph=True, feedback=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = statistics.median(ts)
        points.append({"batch": B, "context": ctx, "step_s": t})
        print(f"B={B:4d} ctx={ctx:5d}: {t * 1e3:.3f} ms", flush=True)
out = {"decoder": spec.name, "weight_bits": spec.weight_bits, "kv_bytes_per_token": spec.kv_bytes_per_token,
       "decode_weight_bytes": spec.decode_weight_bytes(), "gpu": torch.cuda.get_device_name(),
       "how": "CUDA-graph decode step, CUDA events, median of %d; positions = context (all members equal)" % args.reps,
       "points": points}
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
