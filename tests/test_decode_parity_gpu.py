"""End-to-end parity of the shared decode path on the B200 against the CPU oracle.

C1 (BASELINE.json configs[0]): tiny decoder, 2 task prefill
modules + 1 frozen shared decode module, mixed-model batch of 8 prompts
(alternating task), lengths U[16,64] seed 1234, greedy decode 32 steps.

Bars (north_star): logits max-abs <= 2e-2; greedy token sequences bit-exact
wherever the oracle's own decision is not a near-tie (top-2 margin >= 2 x tol).
The greedy check is done two ways: (1) the GPU's free-running sequences must
equal the oracle's free-running sequences for this seeded workload, except a
fork at a step where the oracle's own top-2 margin is < 2x the tolerance;
(2) the oracle re-scores the GPU's history (teacher forcing) and every GPU token must
be the oracle's argmax — or, only where the oracle's own top-2 margin is below
2x the logit tolerance (a near-tie no bf16 implementation can order reliably),
one of the oracle's near-top tokens; the number of such exemptions is reported.
"""
import random

import pytest
import torch

from oracle.decoder_ref import OracleDecoder, OracleSpec, argmax_lowest, greedy_shared_decode, teacher_forced

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2


def oracle_spec(spec):
    return OracleSpec(vocab=spec.vocab, hidden=spec.hidden, n_layers=spec.n_layers, n_q_heads=spec.n_q_heads,
                      n_kv_heads=spec.n_kv_heads, head_dim=spec.head_dim, ffn=spec.ffn,
                      rope_theta=spec.rope_theta, rms_eps=spec.rms_eps, qkv_bias=spec.qkv_bias)


def make_prompts(n, vocab, seed=1234, lo=16, hi=64):
    r = random.Random(seed)
    return [[r.randrange(vocab) for _ in range(r.randint(lo, hi))] for _ in range(n)]


def run_gpu(spec, w_d, w_ps, prompts, module_of, n_steps, cuda, graph=True):
    """GPU SUN pipeline: task prefill modules fill the shared paged pool, then the
    shared decode module decodes the mixed batch greedily."""
    from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
    from paper_2603_02599_b200.modules import PrefillModule, SharedDecodeModule
    from paper_2603_02599_b200.weights import DeviceWeights

    max_ctx = max(len(p) for p in prompts) + n_steps + 1
    B = len(prompts)
    kv = KvPool(spec, num_pages=B * pages_for(max_ctx) + 8, device=cuda)
    kv.tensor.zero_()
    alloc = PageAllocator(kv.num_pages)
    pages = [alloc.alloc(pages_for(len(p) + n_steps)) for p in prompts]
    dec = SharedDecodeModule(spec, DeviceWeights(spec, w_d, cuda, max_ctx), kv, max_batch=B, max_context=max_ctx)
    first = [0] * B
    first_logits = torch.zeros(B, spec.vocab)
    for tau, w_p in enumerate(w_ps):
        pre = PrefillModule(spec, DeviceWeights(spec, w_p, cuda, max_ctx), kv, max_batch=B, max_context=max_ctx,
                            task_id=tau)
        idx = [i for i in range(B) if module_of[i] == tau]
        f, lg = pre.prefill([prompts[i] for i in idx], [pages[i] for i in idx])
        for j, i in enumerate(idx):
            first[i] = f[j]
            first_logits[i] = lg[j].cpu()
    toks = [[f] for f in first]
    bt = torch.zeros(B, dec.max_pages, dtype=torch.int32)
    for i, p in enumerate(pages):
        bt[i, :len(p)] = torch.tensor(p, dtype=torch.int32)
    logits = [first_logits]
    if graph == "host":  # decode_host: persistent pinned buffers, one graph with the copies
        h_tk, h_pos = torch.zeros(B, dtype=torch.int32).pin_memory(), torch.zeros(B, dtype=torch.int32).pin_memory()
        h_bt, h_out = bt.clone().pin_memory(), torch.zeros(B, dtype=torch.int32).pin_memory()
    for t in range(n_steps):
        tk = torch.tensor([x[-1] for x in toks], dtype=torch.int32)
        pos = torch.tensor([len(p) + t for p in prompts], dtype=torch.int32)
        if graph == "host":
            h_tk.copy_(tk)
            h_pos.copy_(pos)
            nxt = dec.decode_host(h_tk, h_pos, h_bt, h_out).clone()
        else:
            nxt = dec.decode(tk, pos, bt, graph=graph).cpu()
        logits.append(dec.logits[:B].cpu().clone())
        for i in range(B):
            toks[i].append(int(nxt[i]))
    # per sequence [1 + n_steps, V]
    return toks, [torch.stack([logits[t][i] for t in range(n_steps + 1)]) for i in range(B)]


def check_parity(spec, w_d, w_ps, prompts, module_of, n_steps, cuda, graph=True, require_free_run=True):
    osp = oracle_spec(spec)
    max_pos = max(len(p) for p in prompts) + n_steps + 1
    o_dec = OracleDecoder(osp, w_d, max_pos)
    o_pre = [OracleDecoder(osp, w, max_pos) for w in w_ps]
    g_toks, g_logits = run_gpu(spec, w_d, w_ps, prompts, module_of, n_steps, cuda, graph)
    tf = teacher_forced(o_pre, o_dec, prompts, module_of, g_toks)
    worst, exempt, total = 0.0, 0, 0
    for i in range(len(prompts)):
        diff = (g_logits[i] - tf[i]).abs().max().item()
        worst = max(worst, diff)
        for t in range(n_steps + 1):
            ol = tf[i][t]
            top = int(argmax_lowest(ol[None])[0])
            total += 1
            if g_toks[i][t] != top:
                top2 = ol.topk(2).values
                margin = (top2[0] - top2[1]).item()
                assert margin < 2 * LOGIT_TOL and ol[top] - ol[g_toks[i][t]] < 2 * LOGIT_TOL, (
                    f"seq {i} step {t}: GPU token {g_toks[i][t]} vs oracle argmax {top} (margin {margin:.4f})")
                exempt += 1
    per_step = [max((g_logits[i][t] - tf[i][t]).abs().max().item() for i in range(len(prompts)))
                for t in range(n_steps + 1)]
    print("per-step logit max-abs:", " ".join(f"{x:.3g}" for x in per_step))
    assert worst <= LOGIT_TOL, f"logits max-abs {worst:.4g} > {LOGIT_TOL}; per step {per_step}"
    # Random-init logits are flat (top-2 gap ~ 0.35 sigma): ~14% of steps have an
    # oracle margin < 2*tol and a bf16 path flips a few of those. Every GPU token
    # is the oracle's argmax except at such near-ties; their rate is bounded here.
    print(f"near-tie exemptions: {exempt}/{total}, logits max-abs {worst:.3g}")
    assert exempt <= max(2, total * 5 // 100), f"{exempt}/{total} near-tie exemptions"
    if require_free_run:
        o_toks, o_logits, o_margins = greedy_shared_decode(o_pre, o_dec, prompts, module_of, n_steps)
        for i in range(len(prompts)):
            if g_toks[i] != o_toks[i]:
                t = next(t for t in range(n_steps + 1) if g_toks[i][t] != o_toks[i][t])
                # teacher forcing above covers every step; a free-running fork is only
                # acceptable where the oracle itself is at a near-tie
                ol = tf[i][t]
                top2 = ol.topk(2).values
                assert (top2[0] - top2[1]).item() < 2 * LOGIT_TOL, f"seq {i} forks at step {t} without a near-tie"
    return worst, exempt, total


@pytest.mark.parametrize("graph", [False, True, "host"])
def test_tiny_mixed_batch_greedy_bit_exact(cuda, graph):
    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import init_weights, perturb

    w_d = init_weights(TINY, seed=0)
    w_ps = [perturb(TINY, w_d, seed=1), perturb(TINY, w_d, seed=2)]
    prompts = make_prompts(8, TINY.vocab)
    check_parity(TINY, w_d, w_ps, prompts, [i % 2 for i in range(8)], 32, cuda, graph)


def test_cluster_chain_shapes_mixed_batch(cuda):
    """8B-wide layer (hidden 4096, 32 q / 8 kv heads of 128) at batch 40: the decode
    step runs the 4-CTA cluster chain with S = 4 DSMEM phases (O, gate_up, down: 32
    tiles) and an S = 2 phase (QKV: 48 tiles), single- and two-chunk owners (bn = 48),
    end to end vs the oracle."""
    from dataclasses import replace

    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import init_weights, perturb

    spec = replace(TINY, name="wide", vocab=1024, hidden=4096, n_layers=1, n_q_heads=32, n_kv_heads=8, head_dim=128,
                   ffn=2048, rope_theta=5e5, lm_head_std=0.0125)
    w_d = init_weights(spec, seed=0)
    w_ps = [perturb(spec, w_d, seed=1), perturb(spec, w_d, seed=2)]
    prompts = make_prompts(40, spec.vocab, lo=8, hi=24)
    check_parity(spec, w_d, w_ps, prompts, [i % 2 for i in range(40)], 8, cuda, graph=True)


def _dequantized_decoder_weights(spec, w):
    """QSUN oracle: θ_d's linear layers as the exact bf16(q * s) operands of SUN-W4."""
    from oracle import quant_ref

    out = dict(w)
    for l in range(spec.n_layers):
        for k in ("wq", "wk", "wv", "wo", "wg", "wu", "wd"):
            q, s = quant_ref.quantize(w[f"l{l}.{k}"])
            out[f"l{l}.{k}"] = quant_ref.dequantize(q, s)
    return out


@pytest.mark.parametrize("variant", ["qsun_w4", "qsun_w4_b12", "qkv_bias"])
def test_tiny_variants_mixed_batch(cuda, variant):
    """QSUN (W4A16 g128 shared decoder, bf16 prefill modules and lm_head,
    PAPER.md:515-519) and Qwen2.5-style QKV bias, end to end vs the oracle."""
    from dataclasses import replace

    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import init_weights, perturb

    if variant.startswith("qsun_w4"):
        spec = replace(TINY, name="tiny-w4", ffn=768, weight_bits=4)  # W4 needs K % 128 == 0
    else:
        spec = replace(TINY, name="tiny-bias", qkv_bias=True)
    w_d = init_weights(spec, seed=0)
    w_ps = [perturb(spec, w_d, seed=1), perturb(spec, w_d, seed=2)]
    n = 12 if variant == "qsun_w4_b12" else 6  # 6 rows: the small-batch W4 GEMV; 12: the W4 chain
    prompts = make_prompts(n, spec.vocab)
    module_of = [i % 2 for i in range(n)]
    if variant.startswith("qsun_w4"):
        # GPU: DeviceWeights quantises θ_d in-kernel; prefill modules stay bf16
        from dataclasses import replace as rp

        spec16 = rp(spec, weight_bits=16)
        check_parity_mixed(spec, spec16, w_d, _dequantized_decoder_weights(spec, w_d), w_ps, prompts, module_of, 16,
                           cuda)
    else:
        check_parity(spec, w_d, w_ps, prompts, module_of, 16, cuda, graph=True)


def check_parity_mixed(spec_dec, spec_pre, w_d, w_d_oracle, w_ps, prompts, module_of, n_steps, cuda):
    """Like check_parity, with distinct decode (e.g. W4) and prefill (bf16) specs."""
    from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
    from paper_2603_02599_b200.modules import PrefillModule, SharedDecodeModule
    from paper_2603_02599_b200.weights import DeviceWeights

    max_ctx = max(len(p) for p in prompts) + n_steps + 1
    B = len(prompts)
    kv = KvPool(spec_pre, num_pages=B * pages_for(max_ctx) + 8, device=cuda)
    kv.tensor.zero_()
    alloc = PageAllocator(kv.num_pages)
    pages = [alloc.alloc(pages_for(len(p) + n_steps)) for p in prompts]
    dec = SharedDecodeModule(spec_dec, DeviceWeights(spec_dec, w_d, cuda, max_ctx), kv, max_batch=B,
                             max_context=max_ctx)
    toks = [[0] for _ in prompts]
    logits = [torch.zeros(B, spec_pre.vocab)]
    for tau, w_p in enumerate(w_ps):
        pre = PrefillModule(spec_pre, DeviceWeights(spec_pre, w_p, cuda, max_ctx), kv, max_batch=B,
                            max_context=max_ctx, task_id=tau)
        idx = [i for i in range(B) if module_of[i] == tau]
        f, lg = pre.prefill([prompts[i] for i in idx], [pages[i] for i in idx])
        for j, i in enumerate(idx):
            toks[i] = [f[j]]
            logits[0][i] = lg[j].cpu()
    bt = torch.zeros(B, dec.max_pages, dtype=torch.int32)
    for i, p in enumerate(pages):
        bt[i, :len(p)] = torch.tensor(p, dtype=torch.int32)
    for t in range(n_steps):
        nxt = dec.decode(torch.tensor([x[-1] for x in toks], dtype=torch.int32),
                         torch.tensor([len(p) + t for p in prompts], dtype=torch.int32), bt).cpu()
        logits.append(dec.logits[:B].cpu().clone())
        for i in range(B):
            toks[i].append(int(nxt[i]))
    osp = oracle_spec(spec_pre)
    o_dec = OracleDecoder(osp, w_d_oracle, max_ctx + 2)
    o_pre = [OracleDecoder(osp, w, max_ctx + 2) for w in w_ps]
    tf = teacher_forced(o_pre, o_dec, prompts, module_of, toks)
    worst, exempt = 0.0, 0
    for i in range(B):
        g = torch.stack([logits[t][i] for t in range(n_steps + 1)])
        worst = max(worst, (g - tf[i]).abs().max().item())
        for t in range(n_steps + 1):
            top = int(argmax_lowest(tf[i][t][None])[0])
            if toks[i][t] != top:
                top2 = tf[i][t].topk(2).values
                assert (top2[0] - top2[1]).item() < 2 * LOGIT_TOL
                exempt += 1
    print(f"mixed-spec parity: logits max-abs {worst:.3g}, near-tie exemptions {exempt}/{B * (n_steps + 1)}")
    assert worst <= LOGIT_TOL, worst
    assert exempt <= max(2, B * (n_steps + 1) * 5 // 100)


@pytest.mark.parametrize("variant", ["tiny", "qkv_bias"])
def test_grouped_prefill_matches_row_prefill(cuda, variant):
    """Token-parallel prefill with row-grouped attention (one CTA stages a prompt's
    KV pages once for up to 16 / G query rows) equals the ungrouped row-per-CTA
    attention: same KV written, same first-token logits (fp32 summation order of
    the warp merge aside)."""
    import random

    from dataclasses import replace

    from paper_2603_02599_b200.kvpool import KvPool, PageAllocator, pages_for
    from paper_2603_02599_b200.modules import PrefillModule
    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import DeviceWeights, init_weights

    spec = TINY if variant == "tiny" else replace(TINY, n_q_heads=10, n_kv_heads=2, qkv_bias=True, name="tiny-bias")
    w = init_weights(spec, seed=5)
    r = random.Random(9)
    prompts = [[r.randrange(spec.vocab) for _ in range(r.randint(20, 70))] for _ in range(5)]
    max_ctx = 80
    out = []
    for grouped in (True, False):
        kv = KvPool(spec, 5 * pages_for(max_ctx) + 2, cuda)
        kv.tensor.zero_()
        alloc = PageAllocator(kv.num_pages)
        pages = [alloc.alloc(pages_for(len(p))) for p in prompts]
        pre = PrefillModule(spec, DeviceWeights(spec, w, cuda, max_ctx), kv, 48, max_ctx, task_id=0, grouped=grouped)
        first, logits = pre.prefill(prompts, pages)
        torch.cuda.synchronize()
        out.append((first, logits.cpu(), kv.tensor.float().cpu(), pages))
    (f0, l0, k0, p0), (f1, l1, k1, p1) = out
    assert p0 == p1
    assert (l0 - l1).abs().max().item() <= 1e-2
    assert (k0 - k1).abs().max().item() <= 2e-2 * max(1.0, k1.abs().max().item())
    for i in range(len(prompts)):
        if f0[i] != f1[i]:  # only a near-tie may flip
            top2 = l1[i].topk(2).values
            assert (top2[0] - top2[1]).item() < 2e-2


def test_decode_host_pipelined_equals_synchronous(cuda):
    """decode_host(sync=False) as bench.py's e2e serving loop drives it — one pinned token
    buffer that is each step's D2H destination and the next step's H2D source, positions
    alternating between two pinned buffers rewritten only after the step two back — ends in
    exactly the state the synchronous host loop reaches: same KV cache, same tokens."""
    from paper_2603_02599_b200.kvpool import KvPool, pages_for
    from paper_2603_02599_b200.modules import SharedDecodeModule
    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import DeviceWeights, init_weights

    spec, B, steps = TINY, 6, 12
    ctx = [5, 17, 30, 2, 44, 21]
    max_ctx = max(ctx) + steps + 8
    dw = DeviceWeights(spec, init_weights(spec, 3), cuda, max_ctx)
    npg = pages_for(max_ctx)
    bt = torch.zeros(B, npg, dtype=torch.int32)
    for i in range(B):
        bt[i] = torch.arange(i * npg, (i + 1) * npg, dtype=torch.int32)
    tok0 = torch.tensor([3, 99, 7, 250, 1, 42], dtype=torch.int32)
    finals = []
    for mode in ("sync", "pipelined"):
        kv = KvPool(spec, B * npg + 2, cuda)
        kv.fill_random_(11)
        dec = SharedDecodeModule(spec, dw, kv, B, max_ctx)
        h_tok, h_bt = tok0.clone().pin_memory(), bt.clone().pin_memory()
        pos = [torch.tensor(ctx, dtype=torch.int32).pin_memory() for _ in range(2)]
        if mode == "sync":
            out = torch.zeros(B, dtype=torch.int32).pin_memory()
            for t in range(steps):
                pos[0].copy_(torch.tensor(ctx, dtype=torch.int32) + t)
                dec.decode_host(h_tok, pos[0], h_bt, out)
                h_tok.copy_(out)
        else:
            evs = [torch.cuda.Event(), torch.cuda.Event()]
            for t in range(steps):
                k = t & 1
                if t >= 2:
                    evs[k].synchronize()
                pos[k].copy_(torch.tensor(ctx, dtype=torch.int32) + t)
                dec.decode_host(h_tok, pos[k], h_bt, h_tok, sync=False)
                evs[k].record()
            torch.cuda.synchronize()
        finals.append((h_tok.clone(), kv.tensor.clone().cpu()))
    assert torch.equal(finals[0][0], finals[1][0])
    assert torch.equal(finals[0][1].view(torch.int16), finals[1][1].view(torch.int16))
