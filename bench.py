#!/usr/bin/env python
"""bench.py — SUN shared-decode throughput on B200 (BASELINE.json metric).

A "step" is one decode step of the frozen shared decode module over the
rank's mixed-model batch (members prefilled by different task modules, routed
to this GPU by the model-agnostic LOT decode router). Default workload = C3:
Llama-3.1-8B-shaped bf16 decoder, 8 task prefill modules with a Zipf(1.5)
request mix (poolsim trace seed 42), 64 sequences per GPU at ISL 1024 /
OSL 256 steady state (contexts 1024..1279). Weights are random-init
(no checkpoints offline) and the KV pages are a seeded on-device fill
(cost excluded; the prefill→decode hand-off is measured separately).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c4|c5|c1]
       [--impl sun|reference] [--routing lot|pinned]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one decode worker
per GPU, weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s/GPU (mixed-model shared decode) at 1/2/4/8 B200; TPOT p50; HBM GB/s"

CONFIGS = {
    "c1": dict(spec="tiny", bits=16, batch=8, isl=48, osl=32, n_models=2, alpha=0.0,
               workload="C1 tiny decoder, 2 task prefill modules + shared decoder, mixed batch 8"),
    "c2": dict(spec="llama3.2-1b", bits=16, batch=64, isl=1984, osl=128, n_models=4, alpha=0.0,
               workload="C2 Llama-3.2-1B-shaped bf16, 4 prefill modules, mixed batch 64, ctx ~2k"),
    "c3": dict(spec="llama3.1-8b", bits=16, batch=64, isl=1024, osl=256, n_models=8, alpha=1.5,
               workload="C3 Llama-3.1-8B-shaped bf16, 8 prefill modules, Zipf a=1.5 mix, 64 seq/GPU, "
                        "ISL 1024 OSL 256 steady state (ctx 1024-1279)"),
    "c4": dict(spec="llama3.1-8b", bits=4, batch=128, isl=4032, osl=128, n_models=8, alpha=1.5,
               workload="C4 QSUN Llama-3.1-8B-shaped W4A16 g128 decoder, batch 128, ctx ~4k"),
    "c5": dict(spec="qwen2.5-14b", bits=16, batch=32, isl=16320, osl=128, n_models=16, alpha=1.5,
               workload="C5 Qwen2.5-14B-shaped bf16, 16 prefill modules, 32 seq/GPU, ctx ~16k",
               cpu_max_batch=4),  # CPU sample: 4 of the 32 sequences (fp32 KV of all 32 is ~200 GB)
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------- workload
def build_assignment(cfg, world, routing):
    """Route B*world requests of the Zipf trace over the decode pool with the
    reference's rules (LOT anticipatory load, or PINNED model i -> worker i%K).
    Returns per-worker lists of (request id, model id)."""
    from paper_2603_02599_b200.router import DecodeDispatcher, PoolSnapshot
    from paper_2603_02599_b200.sun_types import DecodeRule, RoutingPolicy
    from paper_2603_02599_b200.trace import ArrivalProcess, WorkloadSpec, generate_trace

    need = cfg["batch"] * world
    ws = WorkloadSpec(n_models=cfg["n_models"], total_rps=100.0, alpha=cfg["alpha"], isl=cfg["isl"],
                      osl=cfg["osl"], grace_period=0.0, measurement_window=need / 100.0 + 5, drain_margin=0.0,
                      seed=42, arrival_process=ArrivalProcess.DETERMINISTIC)
    trace = generate_trace(ws)[:need]
    n = cfg["n_models"]
    wids = list(range(n, n + world))
    if routing == "pinned":
        disp = DecodeDispatcher(RoutingPolicy(decode_rule=DecodeRule.PINNED),
                                pinned_map={m: wids[m % world] for m in range(n)})
    else:
        disp = DecodeDispatcher(RoutingPolicy(decode_rule=DecodeRule.LEAST_OUTSTANDING_TOKENS))
    load = {w: [0, 0, 0] for w in wids}
    per = {w: [] for w in wids}
    for r in trace:
        pool = [PoolSnapshot(w, load[w][0], load[w][1], load[w][2]) for w in wids]
        w = disp.route(r, pool)
        load[w][1] += r.isl
        load[w][2] += r.target_osl - 1
        per[w].append((r.id, r.model_id))
    return [per[w] for w in wids]


def contexts_for(cfg, nseq):
    """Steady-state continuous batching: members spread evenly over decode progress."""
    return [cfg["isl"] + (j * cfg["osl"]) // max(nseq, 1) for j in range(nseq)]


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- CPU baseline
class CpuOracleStep:
    """The oracle (oracle/decoder_ref.py: CPU fp32, batched linear layers, attention
    per sequence) decoding the workload's mixed batch on the host cores: every
    layer of the decoder, the lm_head and the greedy argmax — one real full-depth
    decode step per call, no extrapolation. KV caches are seeded random at the
    workload's contexts (set up once, not timed)."""

    def __init__(self, cfg, max_batch: int | None = None):
        import torch

        from oracle.decoder_ref import OracleDecoder, OracleSpec
        from paper_2603_02599_b200.spec import SPECS
        from paper_2603_02599_b200.weights import init_weights

        torch.set_num_threads(os.cpu_count() or 1)
        self.threads = torch.get_num_threads()
        spec = SPECS[cfg["spec"]]
        self.spec = spec
        self.B = cfg["batch"] if max_batch is None else min(cfg["batch"], max_batch)
        self.ctx = contexts_for(cfg, self.B)
        osp = OracleSpec(spec.vocab, spec.hidden, spec.n_layers, spec.n_q_heads, spec.n_kv_heads, spec.head_dim,
                         spec.ffn, spec.rope_theta, spec.rms_eps, spec.qkv_bias)
        self.dec = OracleDecoder(osp, init_weights(spec, seed=0), max(self.ctx) + 256)
        g = torch.Generator().manual_seed(7)
        L = spec.n_layers
        self.caches = [{"k": [torch.randn(c, spec.n_kv_heads, spec.head_dim, generator=g) for _ in range(L)],
                        "v": [torch.randn(c, spec.n_kv_heads, spec.head_dim, generator=g) for _ in range(L)]}
                       for c in self.ctx]
        self.toks = [int(x) for x in torch.randint(0, spec.vocab, (self.B,), generator=g)]
        self.i = 0
        part = "" if self.B == cfg["batch"] else f"first {self.B} of "
        self.sample = (f"oracle decode steps of the {part}{cfg['batch']}-sequence mixed batch, all {L} layers + lm_head + "
                       f"argmax (fp32, batched GEMMs, per-sequence attention over ctx "
                       f"{min(self.ctx)}-{max(self.ctx)}), {self.threads} threads")

    def step(self) -> float:
        """Seconds of one full decode step (tokens fed back)."""
        from oracle.decoder_ref import argmax_lowest, decode_batch_layers

        pos = [c + self.i for c in self.ctx]
        self.i += 1
        t0 = time.perf_counter()
        logits = decode_batch_layers(self.dec, self.toks, pos, self.caches, range(self.spec.n_layers))
        self.toks = [int(x) for x in argmax_lowest(logits)]
        return time.perf_counter() - t0


def cpu_baseline(cfg, steps=5, warmup=1):
    """Median of `steps` real full-depth oracle decode steps on the host cores (of the
    first cfg["cpu_max_batch"] sequences where the whole batch's fp32 KV does not fit
    a bounded host sample; tokens/s is then that sample's)."""
    o = CpuOracleStep(cfg, cfg.get("cpu_max_batch"))
    ts = [o.step() for _ in range(warmup + steps)][warmup:]
    t = statistics.median(ts)
    return o.B / t, o.sample + f"; median of {steps} steps after {warmup} warm-up", o.threads, t


def simulator_wall(cfg, n_requests=2000):
    """The restated simulator (scheduler.run = poolsim.engine.run's semantics, golden-
    pinned) serving this config's Zipf trace with the reference's analytic step
    price: wall time and simulated decode steps per second on one host core (SURVEY
    §8(d)(2): it computes no tokens; a reported baseline of the control plane)."""
    from paper_2603_02599_b200 import pricing, scheduler
    from paper_2603_02599_b200.sun_types import ClusterConfig, GpuSpec, ModelProfile, PoolMode, RoutingPolicy
    from paper_2603_02599_b200.trace import ArrivalProcess, WorkloadSpec, generate_trace

    n = cfg["n_models"]
    models = tuple(ModelProfile(model_id=i, param_count=8.03e9, kv_bytes_per_token=131072, shared_decoder=True)
                   for i in range(n))
    cluster = ClusterConfig(models=models, decode_pool_mode=PoolMode.SHARED, decode_pool_size=1,
                            routing_policy=RoutingPolicy(), gpu_spec=GpuSpec.b200())
    cost = pricing.CostParams(prefill_flops_per_token=1.606e10, prefill_fixed_overhead=0.0293,
                              decode_fixed_overhead=0.00543, dequant_compute_penalty=1.242, mfu=0.753, mbu=0.953)
    ws = WorkloadSpec(n_models=n, total_rps=20.0, alpha=cfg["alpha"], isl=cfg["isl"], osl=cfg["osl"],
                      grace_period=0.0, measurement_window=n_requests / 20.0, drain_margin=0.0, seed=42,
                      arrival_process=ArrivalProcess.POISSON)
    trace = generate_trace(ws)
    t0 = time.perf_counter()
    res = scheduler.run(cluster, trace, cost)
    wall = time.perf_counter() - t0
    steps = len(res.log.steps)
    return {"impl": "scheduler.run (restatement of poolsim engine.run, pinned to its golden runs)",
            "requests": len(trace), "decode_steps": steps, "wall_s": wall, "steps_per_s": steps / wall, "cores": 1}


def reference_arm(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    t_setup = time.perf_counter()
    o = CpuOracleStep(cfg, cfg.get("cpu_max_batch"))
    setup_s = time.perf_counter() - t_setup
    for _ in range(args.warmup):
        o.step()
    times = [o.step() for _ in range(args.steps)]
    t = statistics.median(times)
    value = o.B / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "ms_per_step_mean": 1e3 * sum(times) /
        len(times), "timed_s": sum(times), "setup_s": setup_s, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "decoder": o.spec.name, "batch_per_gpu": o.B,
                   "global_batch": o.B, "ctx_min": min(o.ctx), "ctx_max": max(o.ctx), "routing": args.routing,
                   "impl": "CPU oracle port (oracle/decoder_ref.py; the reference computes no tokens)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": o.threads, "kind": "port",
                         "sample": o.sample + f"; median of {args.steps} timed steps"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["simulator_wall"] = simulator_wall(cfg)
    except Exception as e:  # a reported side number: never fail the arm on it
        line["simulator_wall"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- KV hand-off leg (N > 1)
HANDOFF_PAGES = 64  # one C3 request: ISL 1024 = 64 pages of 16 tokens (128 MiB at 8B geometry)


def handoff_local(kv, dev, reps=5):
    """N = 1: the product hand-off path (handoff.copy_pages -> sun_kv_handoff_copy, one
    copy-engine transfer per consecutive page run) between two page runs of this GPU's own
    pool — the same C-ABI call the N > 1 leg makes into a peer's pool over NVLink, here a
    device-to-device copy (reads and writes the same HBM): the per-request overhead and a
    lower bound of the path, not an NVLink figure."""
    import torch

    from paper_2603_02599_b200.handoff import copy_pages

    src = list(range(kv.num_pages - HANDOFF_PAGES, kv.num_pages))
    dst = list(range(kv.num_pages - 2 * HANDOFF_PAGES, kv.num_pages - HANDOFF_PAGES))
    nbytes = HANDOFF_PAGES * kv.page_bytes
    s = torch.cuda.Stream(device=dev)
    dst_struct = kv.struct()
    best = float("inf")
    for i in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        copy_pages(kv, src, dst_struct, dst, s)
        e1.record(s)
        e1.synchronize()
        if i > 0:
            best = min(best, e0.elapsed_time(e1))
    return {"bytes_per_request": nbytes, "pages": HANDOFF_PAGES, "transport": "same-device copy engine (D2D)",
            "ms_per_request": best, "GB_s": nbytes / (best / 1e3) / 1e9}


def handoff_leg(kv, rank, world, dev, spec, reps=5):
    """Every rank hands one ISL-1024 request's KV (the last HANDOFF_PAGES pages of its
    pool, reserved for this) to rank + 1 at the same time, two ways: (1) the
    product path, a CUDA-IPC peer copy into the receiver's pages on the copy engines
    (handoff.copy_pages: NVLink 5 / NVSwitch), (2) NCCL send/recv of the same bytes.
    Device-timed (CUDA events), after the decode timing; returns per-transport GB/s
    (min / mean over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2603_02599_b200.handoff import RemotePool, copy_pages, export_pool

    ctrl = dist.new_group(backend="gloo")
    mine = export_pool(kv)
    allh = [None] * world
    dist.all_gather_object(allh, mine.numpy().tobytes(), group=ctrl)
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    remote = RemotePool(torch.frombuffer(bytearray(allh[nxt]), dtype=torch.uint8))
    src = list(range(kv.num_pages - HANDOFF_PAGES, kv.num_pages))
    dst = list(range(remote.num_pages - HANDOFF_PAGES, remote.num_pages))
    nbytes = HANDOFF_PAGES * kv.page_bytes
    s = torch.cuda.Stream(device=dev)
    out = {"bytes_per_request": nbytes, "pages": HANDOFF_PAGES}

    def timed(fn):
        for i in range(reps + 1):
            dist.barrier(group=ctrl)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            if i == 0:
                best = float("inf")  # first rep warms the mapping / NCCL channels
            else:
                best = min(best, e0.elapsed_time(e1))
        return best

    ms = timed(lambda: copy_pages(kv, src, remote.struct, dst, s))
    buf = torch.empty((HANDOFF_PAGES,) + tuple(kv.tensor.shape[1:]), dtype=kv.tensor.dtype, device=dev)

    def nccl():
        with torch.cuda.stream(s):
            ops = [dist.P2POp(dist.isend, kv.tensor[src[0]:src[0] + HANDOFF_PAGES], nxt),
                   dist.P2POp(dist.irecv, buf, prv)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    ms_nccl = timed(nccl)
    gb = torch.tensor([nbytes / (ms / 1e3) / 1e9, nbytes / (ms_nccl / 1e3) / 1e9], device=dev)
    lo, tot = gb.clone(), gb.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(tot)
    remote.close()
    out["peer_copy"] = {"gbps_min": float(lo[0]), "gbps_mean": float(tot[0]) / world,
                        "transport": "CUDA IPC peer copy on the copy engines (sun_kv_handoff_copy)"}
    out["nccl_p2p"] = {"gbps_min": float(lo[1]), "gbps_mean": float(tot[1]) / world,
                       "transport": "NCCL send/recv (handoff.send_kv path)"}
    out["pattern"] = "every rank sends one request to rank+1 simultaneously; best of 5 after 1 warm-up"
    return out


# --------------------------------------------------------------------------- GPU arm
def kernel_bytes(spec, B, ctx):
    """Algorithmic bytes per launch of each kernel class (SURVEY.md §8(d) terms)."""
    h, d = spec.hidden, spec.head_dim
    qd, kd, f, V = spec.n_q_heads * d, spec.n_kv_heads * d, spec.ffn, spec.vocab

    def wbytes(rows, k):
        return rows * k // 2 + rows * (k // spec.group_size) * 2 if spec.weight_bits == 4 else rows * k * 2

    kv_layer = sum(c + 1 for c in ctx) * 2 * kd * 2
    return {
        "gemm_qkv_rope_kv": wbytes(qd + 2 * kd, h) + B * h * 2 + B * (qd + 2 * kd) * 2,
        "attention": kv_layer + B * qd * 2 + B * spec.n_q_heads * 8,
        "attn_combine": B * qd * 2,
        "gemm_o_resid_norm": wbytes(h, qd) + B * qd * 2 + B * h * 10,
        "gemm_gate_up_swiglu": wbytes(2 * f, h) + B * h * 2 + B * f * 2,
        "gemm_down_resid_norm": wbytes(h, f) + B * f * 2 + B * h * 10,
        "gemm_lm_head_argmax": V * h * 2 + B * h * 2 + B * V * 4,
        "embed_norm": B * h * 8,
        "argmax": 0,
        # SUN_GEMM_CHAIN=1: O + gate_up + down + the next layer's QKV in one launch
        "gemm_chain": (wbytes(h, qd) + wbytes(2 * f, h) + wbytes(h, f) + wbytes(qd + 2 * kd, h)
                       + B * (qd + h + f + h) * 2 + B * h * 20 + B * (qd + 2 * kd) * 2),
    }


def gpu_arm(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2603_02599_b200.kvpool import KvPool, pages_for
    from paper_2603_02599_b200.modules import SharedDecodeModule, launch_count
    from paper_2603_02599_b200.pricing import step_bytes
    from paper_2603_02599_b200.spec import SPECS
    from paper_2603_02599_b200.weights import DeviceWeights, init_weights

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = SPECS[cfg["spec"]].with_bits(cfg["bits"]) if cfg["bits"] == 4 else SPECS[cfg["spec"]]
    assign = build_assignment(cfg, world, args.routing)
    mine = assign[rank]
    # PINNED at N > 1 with a Zipf mix can hand one worker more requests than one
    # decode step holds (the kernels take B <= 256): that worker decodes its first
    # 256 (the partitioned baseline is then capacity-bound, as in the paper)
    batch_cap = 256
    capped = len(mine) > batch_cap
    mine = mine[:batch_cap]
    B = len(mine)
    ctx = contexts_for(cfg, B)
    total_steps = args.warmup + args.steps
    max_ctx = max(ctx) + total_steps + args.steps + 8

    t0 = time.perf_counter()
    w = init_weights(spec, seed=0, device=dev)
    dw = DeviceWeights(spec, w, dev, max_ctx, free_source=True)
    del w
    kv = KvPool(spec, sum(pages_for(c + total_steps + args.steps + 2) for c in ctx) + 4 + 2 * HANDOFF_PAGES, dev)
    kv.fill_random_(seed=1000 + rank)
    dec = SharedDecodeModule(spec, dw, kv, max_batch=B, max_context=max_ctx, use_pdl=not args.no_pdl)
    # block tables: contiguous page runs per member
    bt = torch.zeros(B, dec.max_pages, dtype=torch.int32)
    nxt = 0
    for i, c in enumerate(ctx):
        n = pages_for(c + total_steps + args.steps + 2)
        bt[i, :n] = torch.arange(nxt, nxt + n, dtype=torch.int32)
        nxt += n
    g = torch.Generator().manual_seed(11 + rank)
    tokens0 = torch.randint(0, spec.vocab, (B,), generator=g, dtype=torch.int32)
    dec.block_tables[:B].copy_(bt.to(dev))
    dec.tokens[:B].copy_(tokens0.to(dev))
    dec.positions[:B].copy_(torch.tensor(ctx, dtype=torch.int32).to(dev))
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0

    graph = not args.no_graph
    for _ in range(args.warmup):
        dec.step_static(B, args.pps, graph=graph, feedback=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record()
    for i in range(args.steps):
        dec.step_static(B, args.pps, graph=graph, feedback=True)
        evs[i + 1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    t_max = torch.tensor([total_ms], device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_max = float(t_max.item())
    tok_total = B * args.steps
    tok_all = torch.tensor([float(tok_total)], device=dev)
    if world > 1:
        dist.all_reduce(tok_all)
    value = float(tok_all.item()) / (t_max / 1e3)

    # launches inside the timed region: graph replays do not pass through the
    # library's host launch counter, so count the kernels of one captured step
    prof = dec.profile(dec.tokens, dec.positions, dec.block_tables, B, dec.next_tokens, None, args.pps)
    names = dec.kernel_names(batch=B)
    if len(names) != len(prof):  # unsplit attention: no combine launches
        names = dec.kernel_names(combine=False, batch=B)
    per_step_launches = len(names)
    gpu_launches = per_step_launches * args.steps

    # ---- per-kernel attribution (serialised, events after every launch) ----
    pos_now = [c + args.warmup + args.steps for c in ctx]
    by = {}
    for n_, ms in zip(names, prof):
        t = by.setdefault(n_, [0.0, 0])
        t[0] += ms
        t[1] += 1
    kb = kernel_bytes(spec, B, pos_now)
    prof_total = sum(prof)
    dominant = max((k for k in by if k in kb), key=lambda k: by[k][0])
    dom_ms = by[dominant][0] / by[dominant][1]
    peak, peak_kind = load_peaks()
    achieved = kb[dominant] / (dom_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(args.config, {}).get(dominant)
    except Exception:
        pass
    ms_step = t_max / args.steps
    sb = step_bytes(spec, [c + args.warmup for c in ctx])
    step_gbs = sb / (ms_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        pin = lambda t: t.pin_memory()  # noqa: E731
        h_tok = pin(tokens0.clone())
        h_bt = pin(bt.clone())
        # the same contexts as the device-timed loop (its first step's positions; the warm
        # calls below re-run the two before them): the KV those steps wrote is rewritten, and
        # e2e and `value` time the same work
        h_pos = pin(torch.tensor([c + args.warmup - 2 for c in ctx], dtype=torch.int32))
        out = pin(torch.zeros(B, dtype=torch.int32))
        for i in range(2):  # warm (the first call also captures the host-copy graph)
            if graph:
                dec.decode_host(h_tok, h_pos, h_bt, out, pages_per_split=args.pps)
            else:
                dec.decode(h_tok, h_pos, h_bt, pages_per_split=args.pps, graph=False)
                out.copy_(dec.next_tokens[:B])
            h_pos += 1
        # serving-loop pipelining (graph path): one pinned token buffer is both a step's D2H
        # destination and the next step's H2D source (stream-ordered), positions alternate
        # between two pinned buffers whose rewrite waits for the step two back, so the GPU
        # runs a step ahead of the host instead of idling through a sync + relaunch per step
        h_pos2 = [h_pos, pin(h_pos.clone())]
        evs = [torch.cuda.Event(), torch.cuda.Event()]
        if graph:
            h_tok.copy_(out)
            for k in range(2):  # capture both (tokens == out) graphs
                h_pos2[k].copy_(h_pos)
                dec.decode_host(h_tok, h_pos2[k], h_bt, h_tok, pages_per_split=args.pps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        pos_base = h_pos.clone()
        te = time.perf_counter()
        for i in range(args.steps):
            if graph and args.e2e_sync:  # (A/B: synchronise every step, host feedback)
                dec.decode_host(h_tok, h_pos2[0], h_bt, h_tok, pages_per_split=args.pps)
                torch.add(pos_base, i + 1, out=h_pos2[0])
            elif graph:  # H2D inputs + step + D2H next tokens as one graph launch per step
                k = i & 1
                if i >= 2:
                    evs[k].synchronize()  # the step that last read h_pos2[k] is done
                torch.add(pos_base, i, out=h_pos2[k])
                dec.decode_host(h_tok, h_pos2[k], h_bt, h_tok, pages_per_split=args.pps, sync=False)
                evs[k].record()
            else:
                nt = dec.decode(h_tok, h_pos, h_bt, pages_per_split=args.pps, graph=False)
                out.copy_(nt)  # D2H read of the step's result (synchronises)
                h_tok.copy_(out)
                h_pos += 1
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - te
        t_e = torch.tensor([e2e_s], device=dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e = {"value": float(tok_all.item()) / float(t_e.item()), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h_tok.numel() * 4 + h_pos.numel() * 4 + h_bt.numel() * 4),
               "d2h_bytes_per_step": int(out.numel() * 4),
               "api": ("SharedDecodeModule.decode_host(pinned tokens/positions/block_tables) -> pinned next tokens, "
                       "one graph per step (H2D inputs, step, D2H next tokens); the next step's tokens are "
                       "H2D'd from the pinned buffer the previous D2H filled, the host keeps one step ahead"
                       if graph else "SharedDecodeModule.decode(host pinned tokens/positions/block_tables) -> next tokens")}

    handoff = None
    if world > 1 and not args.no_handoff:
        handoff = handoff_leg(kv, rank, world, dev, spec)
    elif not args.no_handoff:
        handoff = handoff_local(kv, dev)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        v, sample, threads, _ = cpu_baseline(cfg, steps=5, warmup=1)
        cpu = {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if spec.weight_bits == 16 else "bf16 act / int4 weight",
            "data": "synthetic: random-init weights N(0,0.02) seed 0, seeded on-device KV fill, poolsim Zipf trace seed 42",
            "config": {"workload": cfg["workload"], "decoder": spec.name, "batch_per_gpu": B,
                       "global_batch": int(tok_all.item()) // args.steps, "ctx_min": min(ctx), "ctx_max": max(ctx),
                       "routing": args.routing, "parallelism": f"{world} shared decode workers (request-level DP)",
                       "models_in_batch": sorted({m for _, m in mine}), "cuda_graph": graph,
                       "rank0_batch_capped_at_256": capped,
                       "pdl": not args.no_pdl,
                       "l2": "inputs larger than L2 (weights + KV per step >> 126 MB), no explicit flush"},
            "tokens_per_s_per_gpu": value / world,
            "tpot_ms_p50": statistics.median(step_ms),
            "hbm_gbps_step": step_gbs,
            "step_bytes": sb,
            "step_roofline_frac": step_gbs / peak,
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "bytes_per_launch": kb[dominant], "avg_launch_ms": dom_ms},
            "kernel_ms_per_step": {k: round(v[0], 4) for k, v in sorted(by.items(), key=lambda x: -x[1][0])},
            "kernel_share": {k: round(v[0] / prof_total, 4) for k, v in by.items()},
            "serialised_step_ms": prof_total,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": gpu_launches,
            "setup_s": setup_s,
            "handoff": handoff,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dry_run_arm(args, cfg):
    """The N-rank bench path without a GPU (gloo, CPU): the same LOT / PINNED routing
    of the Zipf trace over the ranks, a stand-in step of fixed cost per row, the
    barrier + max-over-ranks timing all-reduce and the JSON line. For CPU tests of
    the multi-rank plumbing (tests/test_bench_ranks.py); reports nothing about a GPU."""
    import torch
    import torch.distributed as dist

    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group("gloo")
    mine = build_assignment(cfg, world, args.routing)[rank][:256]
    B = len(mine)
    for _ in range(args.warmup):
        time.sleep(1e-5 * B)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(1e-5 * B)  # stand-in step
    t = torch.tensor([time.perf_counter() - t0])
    tok = torch.tensor([float(B * args.steps)])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tok)
    gathered = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, sorted({m for _, m in mine}))
    else:
        gathered = [sorted({m for _, m in mine})]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": float(tok) / float(t), "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(t) * 1e3 / args.steps,
                          "higher_is_better": True, "scaling": "weak", "dry_run": True,
                          "config": {"workload": cfg["workload"], "batch_per_gpu": B,
                                     "global_batch": int(float(tok)) // args.steps, "routing": args.routing,
                                     "models_per_rank": gathered,
                                     "parallelism": f"{world} shared decode workers (request-level DP)"}}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: start the N ranks ourselves, the way the
    driver does (torch.distributed.run, one process per GPU, 127.0.0.1 rendezvous)."""
    import socket
    import subprocess

    if not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="sun", choices=["sun", "reference"])
    ap.add_argument("--routing", default="lot", choices=["lot", "pinned"])
    ap.add_argument("--pps", type=int, default=0, help="attention pages per split (0 = auto)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-handoff", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo run of the rank plumbing (tests)")
    ap.add_argument("--e2e-sync", action="store_true", help="e2e: synchronise every step (A/B of the pipelining)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_ranks(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    if args.impl == "reference":
        reference_arm(args, cfg)
    elif args.dry_run:
        dry_run_arm(args, cfg)
    else:
        gpu_arm(args, cfg)


if __name__ == "__main__":
    main()
