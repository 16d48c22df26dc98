"""Device-side timeline of one decode step (GEMM + attention launches, PDL on):
earliest CTA start / latest CTA end per launch, gaps between launches."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2603_02599_b200 import _lib
from paper_2603_02599_b200.kvpool import KvPool, pages_for
from paper_2603_02599_b200.modules import SharedDecodeModule
from paper_2603_02599_b200.spec import SPECS
from paper_2603_02599_b200.weights import DeviceWeights, init_weights

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--layers", type=int, default=3, help="layers to print")
ap.add_argument("--stamp", type=int, default=-1, help="launch index whose per-CTA phases to print")
ap.add_argument("--slow", type=int, default=0, help="with --stamp: also list the N CTAs that finish last")
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
max_ctx = max(ctx) + 64
dw = DeviceWeights(spec, init_weights(spec, 0, dev), dev, max_ctx, free_source=True)
kv = KvPool(spec, sum(pages_for(c + 40) for c in ctx) + 4, dev)
kv.fill_random_(1)
dec = SharedDecodeModule(spec, dw, kv, B, max_ctx)
nxt = 0
for i, c in enumerate(ctx):
    n = pages_for(c + 40)
    dec.block_tables[i, :n] = torch.arange(nxt, nxt + n, dtype=torch.int32, device=dev)
    nxt += n
dec.positions[:B] = torch.tensor(ctx, dtype=torch.int32, device=dev)
for _ in range(5):
    dec.step_static(B, 0, graph=False)
cap = 8 * spec.n_layers + 8
lib = _lib.load()
names = ["qkv", "attn", "o", "gate_up", "down"]
for rep in range(2):
    st = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    tl = torch.zeros(cap, 2, dtype=torch.int64, device=dev)
    tl[:, 0] = torch.iinfo(torch.int64).max
    n = ctypes.c_int32()
    torch.cuda.synchronize()
    _lib.check(lib.sun_decode_step_timeline(dec._h, dec.tokens.data_ptr(), dec.positions.data_ptr(),
                                            dec.block_tables.data_ptr(), dec.block_tables.stride(0), B, 0,
                                            dec.next_tokens.data_ptr(), torch.cuda.current_stream().cuda_stream,
                                            tl.data_ptr(), cap, ctypes.byref(n), st.data_ptr() if args.stamp >= 0 else None,
                                            args.stamp), "timeline")
    torch.cuda.synchronize()
t = tl[: n.value].cpu().double()
t0 = t[:, 0].min()
t = (t - t0) / 1e3
short = {"gemm_qkv_rope_kv": "qkv", "attention": "attn", "gemm_o_resid_norm": "o", "gemm_gate_up_swiglu": "gate_up",
         "gemm_down_resid_norm": "down", "gemm_chain": "chain", "gemm_lm_head_argmax": "lm_head"}
lab = [short[k] for k in dec.kernel_names(combine=False, batch=B) if k in short]  # the launches that record a timeline slot
assert len(lab) == n.value, (len(lab), n.value)
print(f"{args.config}: {n.value} launches, step span {t[:, 1].max():.1f} us")
tot = {}
prev_end = 0.0
for i in range(n.value):
    s, e = float(t[i, 0]), float(t[i, 1])
    d = tot.setdefault(lab[i], [0.0, 0.0, 0])
    d[0] += e - max(s, prev_end)   # exclusive time: from previous end (or own start) to own end
    d[1] += e - s
    d[2] += 1
    if i < (len(lab) - 1) * args.layers // spec.n_layers or i == n.value - 1:
        print(f"  {i:3d} {lab[i]:8s} start {s:9.2f} end {e:9.2f} dur {e - s:7.2f} after-prev-end {e - prev_end:7.2f} (overlap {prev_end - s:6.2f})")
    prev_end = max(prev_end, e)
print("per class: exclusive us/launch (end - previous end), inclusive us/launch (end - start)")
for k, (ex, inc, c) in tot.items():
    print(f"  {k:8s} excl {ex / c:7.2f}  incl {inc / c:7.2f}  x{c}")

if args.stamp >= 0:
    sv = st.view(4096, 16).cpu().double()
    sv = sv[sv[:, 0] > 0]
    rel = (sv - t0) / 1e3
    print(f"launch {args.stamp} ({lab[args.stamp]}): {len(sv)} CTAs; phase times relative to step start (us)")
    nm = ["start", "setup", "first_stage", "last_mma", "first_acc", "epi_done", "exit", "-", "parked", "sync1",
          "reduced", "epi_chunk", "qkv_bar1", "qkv_bar2", "qkv_loads"]
    if lab[args.stamp] == "chain":  # per phase (O, gate_up, down, next QKV)
        nm = [f"{ph}:{ev}" for ph in ("o", "gate_up", "down", "qkv") for ev in ("x_ready", "first_mma", "last_mma", "epi_done")]
        if os.environ.get("SEG_STAMPS"):  # -DSUN_W4_SEG_STAMPS build: O-phase segment epilogue split in slots 12..15
            nm[12:16] = ["o:seg_start", "o:parked", "o:peers_in", "o:reduced+epi"]
    for i, name in enumerate(nm):
        if name == "-" or (sv[:, i] == 0).all():
            continue
        c = rel[:, i][sv[:, i] > 0]
        print(f"   {name:12s} min {c.min():9.2f} med {c.median():9.2f} max {c.max():9.2f}")
    if args.slow > 0:
        order = torch.argsort(rel[:, 6], descending=True)[: args.slow]
        print(f"   slowest {args.slow} CTAs (blockIdx: start first_stage last_mma parked sync1 reduced epi_chunk exit)")
        allrows = (st.view(4096, 16)[:, 0] > 0).nonzero().flatten().cpu()
        for k in order.tolist():
            r = rel[k]
            print(f"   {int(allrows[k]):4d}: " + " ".join(f"{float(r[i]):8.2f}" for i in (0, 2, 3, 8, 9, 10, 11, 6)))
