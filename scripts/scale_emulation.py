"""Shared vs per-model-partitioned decode at N = 1, 2, 4, 8 decode GPUs, emulated on
one B200: every rank's batch (from the reference router: LOT for the shared pool,
PINNED model i -> worker i mod N for the partitioned baseline, bench.build_assignment)
is timed here with the real decode step (CUDA graph, C3 steady-state contexts); the
N-GPU step time is the slowest rank's, so TPOT and whole-job tokens/s follow without a
multi-GPU box (each rank is an independent decode worker: no collective on the path).

  python scripts/scale_emulation.py --out profiles/r01/scale_emulation_c3.json
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_02599_b200.kvpool import KvPool, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", required=True)
ap.add_argument("--cap", type=int, default=256, help="per-GPU batch cap (KV capacity of one B200)")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
spec = SPECS[cfg["spec"]]
dev = torch.device("cuda")
B_max = args.cap
ctx_max = cfg["isl"] + cfg["osl"] + 8
dw = DeviceWeights(spec, init_weights(spec, 0, dev), dev, ctx_max + args.reps + 8, free_source=True)
kv = KvPool(spec, B_max * pages_for(ctx_max + args.reps + 8) + 4, dev)
kv.fill_random_(1)
dec = SharedDecodeModule(spec, dw, kv, B_max, ctx_max + args.reps + 8)
n = pages_for(ctx_max + args.reps + 8)
for i in range(B_max):
    dec.block_tables[i, :n] = torch.arange(i * n, (i + 1) * n, dtype=torch.int32, device=dev)
cache = {}


def step_ms(B):
    if B in cache:
        return cache[B]
    ctx = bench.contexts_for(cfg, B)
    dec.positions[:B] = torch.tensor(ctx, dtype=torch.int32, device=dev)
    for _ in range(3):
        dec.step_static(B, 0, graph=True)
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dec.step_static(B, 0, graph=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    cache[B] = statistics.median(ts)
    return cache[B]


rows = []
for routing in ("lot", "pinned"):
    for world in (1, 2, 4, 8):
        full = [len(p) for p in bench.build_assignment(cfg, world, routing)]
        per = [min(b, B_max) for b in full]
        t = [step_ms(B) for B in per]
        tpot = max(t)
        rows.append({"routing": routing, "n_gpus": world, "requests_per_rank": full, "batch_per_rank": per,
                     "step_ms_per_rank": t,
                     "tpot_ms": tpot, "tokens_per_s": sum(per) / (tpot / 1e3)})
        print(f"{routing:6s} N={world}: batches {per} -> TPOT {tpot:.3f} ms, {sum(per) / tpot * 1e3:.0f} tok/s", flush=True)
base = rows[0]["tokens_per_s"]
for r in rows:
    r["speedup_vs_1gpu_lot"] = r["tokens_per_s"] / base
out = {"config": cfg["workload"], "batch_cap": B_max, "how": "each rank's batch timed on one B200 (CUDA graph, median of %d); N-GPU step = "
       "slowest rank (independent decode workers, no collective)" % args.reps, "rows": rows}
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
