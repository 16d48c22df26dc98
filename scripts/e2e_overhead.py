"""Where the C3 e2e step's overhead over the device-timed step goes: per-step wall time of
(a) the device-resident CUDA-graph step launched + synchronised one at a time, (b) the same
with on-device feedback but no per-step sync, (c) SharedDecodeModule.decode_host (H2D inputs
+ step + D2H next tokens as one graph, synchronised)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_02599_b200.kvpool import KvPool, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

cfg = bench.CONFIGS["c3"]
spec = SPECS[cfg["spec"]]
dev = torch.device("cuda")
B = cfg["batch"]
ctx = bench.contexts_for(cfg, B)
N = 50
max_ctx = max(ctx) + 3 * N + 64
dw = DeviceWeights(spec, init_weights(spec, 0, dev), dev, max_ctx, free_source=True)
kv = KvPool(spec, sum(pages_for(c + 3 * N + 40) for c in ctx) + 4, dev)
kv.fill_random_(1)
dec = SharedDecodeModule(spec, dw, kv, B, max_ctx)
npg = pages_for(max(ctx) + 3 * N + 40)
bt = torch.zeros(B, npg, dtype=torch.int32)
nxt = 0
for i, c in enumerate(ctx):
    n = pages_for(c + 3 * N + 40)
    bt[i, :n] = torch.arange(nxt, nxt + n, dtype=torch.int32)
    nxt += n
dec.block_tables[:B, :npg] = bt.to(dev)
dec.positions[:B] = torch.tensor(ctx, dtype=torch.int32, device=dev)
for _ in range(3):
    dec.step_static(B, 0, graph=True, feedback=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    dec.step_static(B, 0, graph=True, feedback=True)
torch.cuda.synchronize()
a = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    dec.step_static(B, 0, graph=True, feedback=True)
    torch.cuda.current_stream().synchronize()
b = (time.perf_counter() - t0) / N
h_tok = torch.zeros(B, dtype=torch.int32).pin_memory()
h_pos = torch.tensor([c + 2 * N for c in ctx], dtype=torch.int32).pin_memory()
h_bt = bt.pin_memory()
out = torch.zeros(B, dtype=torch.int32).pin_memory()
for _ in range(3):
    dec.decode_host(h_tok, h_pos, h_bt, out)
    h_pos += 1
t0 = time.perf_counter()
for _ in range(N):
    dec.decode_host(h_tok, h_pos, h_bt, out)
    h_tok.copy_(out)
    h_pos += 1
c = (time.perf_counter() - t0) / N
print(f"back-to-back graph steps {a*1e3:.3f} ms | one step + sync {b*1e3:.3f} ms | decode_host e2e {c*1e3:.3f} ms")
