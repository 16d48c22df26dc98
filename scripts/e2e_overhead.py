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
N = 40
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

# (d) the pipelined serving loop bench.py's e2e uses: one pinned token buffer as D2H
# destination and next H2D source, positions double-buffered behind events
h_tok2 = torch.zeros(B, dtype=torch.int32).pin_memory()
pos2 = [torch.tensor([c + 3 * N for c in ctx], dtype=torch.int32).pin_memory() for _ in range(2)]
for k in range(2):
    dec.decode_host(h_tok2, pos2[k], h_bt, h_tok2)
evs = [torch.cuda.Event(), torch.cuda.Event()]
base = pos2[0].clone()
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    k = i & 1
    if i >= 2:
        evs[k].synchronize()
    torch.add(base, i, out=pos2[k])
    dec.decode_host(h_tok2, pos2[k], h_bt, h_tok2, sync=False)
    evs[k].record()
torch.cuda.synchronize()
d = (time.perf_counter() - t0) / N
print(f"pipelined decode_host {d*1e3:.3f} ms")

# (e) the same pipelining with the copies issued as separate async memcpys around the
# kernels-only step graph (no memcpy nodes inside the graph)
for k in range(2):
    torch.add(base, 2 * N + k, out=pos2[k])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    k = i & 1
    if i >= 2:
        evs[k].synchronize()
    torch.add(base, 2 * N + i, out=pos2[k])
    dec.tokens[:B].copy_(h_tok2, non_blocking=True)
    dec.positions[:B].copy_(pos2[k], non_blocking=True)
    dec.block_tables[:B, :npg].copy_(h_bt, non_blocking=True)
    dec.step_static(B, 0, graph=True, feedback=False)
    h_tok2.copy_(dec.next_tokens[:B], non_blocking=True)
    evs[k].record()
torch.cuda.synchronize()
e = (time.perf_counter() - t0) / N
print(f"pipelined separate copies {e*1e3:.3f} ms")

# (f) as (e) with a full-width block table (contiguous destination rows) and (g) without
# the block-table copy at all
h_btf = torch.zeros(B, dec.max_pages, dtype=torch.int32)
h_btf[:, :npg] = bt
h_btf = h_btf.pin_memory()
for variant in ("f", "g"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N):
        k = i & 1
        if i >= 2:
            evs[k].synchronize()
        torch.add(base, 3 * N + i, out=pos2[k])
        dec.tokens[:B].copy_(h_tok2, non_blocking=True)
        dec.positions[:B].copy_(pos2[k], non_blocking=True)
        if variant == "f":
            dec.block_tables[:B].copy_(h_btf, non_blocking=True)
        dec.step_static(B, 0, graph=True, feedback=False)
        h_tok2.copy_(dec.next_tokens[:B], non_blocking=True)
        evs[k].record()
    torch.cuda.synchronize()
    print(f"({variant}) {(time.perf_counter() - t0) / N * 1e3:.3f} ms")
