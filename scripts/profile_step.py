"""Run N decode steps of a bench config without CUDA graphs (for ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_02599_b200.kvpool import KvPool, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--no-pdl", action="store_true")
ap.add_argument("--batch", type=int, default=0, help="override the config's batch")
ap.add_argument("--isl", type=int, default=0, help="override the config's context start")
args = ap.parse_args()
cfg = dict(bench.CONFIGS[args.config])
if args.batch:
    cfg["batch"] = args.batch
if args.isl:
    cfg["isl"] = args.isl
spec = SPECS[cfg["spec"]].with_bits(4) if cfg["bits"] == 4 else SPECS[cfg["spec"]]
dev = torch.device("cuda")
B = cfg["batch"]
ctx = bench.contexts_for(cfg, B)
max_ctx = max(ctx) + args.steps + 16
dw = DeviceWeights(spec, init_weights(spec, 0, dev), dev, max_ctx, free_source=True)
kv = KvPool(spec, sum(pages_for(c + args.steps + 4) for c in ctx) + 4, dev)
kv.fill_random_(1)
dec = SharedDecodeModule(spec, dw, kv, B, max_ctx, use_pdl=not args.no_pdl)
nxt = 0
for i, c in enumerate(ctx):
    n = pages_for(c + args.steps + 4)
    dec.block_tables[i, :n] = torch.arange(nxt, nxt + n, dtype=torch.int32, device=dev)
    nxt += n
dec.positions[:B] = torch.tensor(ctx, dtype=torch.int32, device=dev)
for _ in range(args.steps):
    dec.step_static(B, 0, graph=False, feedback=True)
torch.cuda.synchronize()
print("done", len(dec.kernel_names(batch=B)), "kernels/step")
