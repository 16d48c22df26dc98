"""Kernel-level numerics on the B200: each sm_100a kernel vs a plain torch fp32
restatement of the same op on the same inputs (tolerances stated inline)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _r16(b):
    return (b + 15) // 16 * 16


@pytest.mark.parametrize(
    "n_out,k,batch",
    [(256, 256, 1), (768, 256, 8), (1408, 256, 17), (300, 688, 5), (4096, 4096, 64), (6144, 4096, 64),
     (1000, 512, 256), (4096, 14336, 33), (512, 128, 128),
     # more tiles than SMs, not a multiple of 148: stream-K (partial tiles + owner fix-up)
     (28672, 4096, 64), (20000, 512, 40), (128256, 256, 8)],
)
def test_gemm_bf16_matches_fp32(cuda, n_out, k, batch):
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(n_out * 7 + k + batch)
    w = (torch.randn(n_out, k, generator=g) * 0.02).to(torch.bfloat16).to(cuda)
    x = torch.randn(_r16(batch), k, generator=g).to(torch.bfloat16).to(cuda)
    x[batch:] = float("nan")  # padded batch rows must not leak into valid columns
    out = kernels.gemm_bf16(w, x, batch)
    ref = x[:batch].float() @ w.float().t()
    torch.cuda.synchronize()
    # fp32 accumulation of bf16 products: only summation order differs
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))
    # accumulate mode adds onto the existing buffer
    out2 = kernels.gemm_bf16(w, x, batch, out=out.clone(), accumulate=True)
    torch.testing.assert_close(out2, 2 * ref, rtol=1e-4, atol=2e-4 * math.sqrt(k))


def test_gemm_deterministic_split_k(cuda):
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(3)
    w = (torch.randn(4096, 14336, generator=g) * 0.02).to(torch.bfloat16).to(cuda)
    x = torch.randn(64, 14336, generator=g).to(torch.bfloat16).to(cuda)
    a = kernels.gemm_bf16(w, x, 64)
    b = kernels.gemm_bf16(w, x, 64)
    assert torch.equal(a, b)


def test_gemm_deterministic_stream_k(cuda):
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(4)
    w = (torch.randn(28672, 4096, generator=g) * 0.02).to(torch.bfloat16).to(cuda)
    x = torch.randn(64, 4096, generator=g).to(torch.bfloat16).to(cuda)
    a = kernels.gemm_bf16(w, x, 64)
    for _ in range(3):
        assert torch.equal(a, kernels.gemm_bf16(w, x, 64))


@pytest.mark.parametrize("sched", ["0", "2", "vcl2", "novcl", "push", "nochain", "l2chain", "nogemv", "gvchain",
                                   "tileready", "gvcluster", "gvbal0", "gvbal2", "attntile"])
def test_gemm_schedules_subprocess(sched):
    """The GEMM kernel tests and the end-to-end decode parity under the other
    schedules: 0 = cluster split-K / whole tiles only, 2 = stream-K on every
    GEMM whose partials fit (covers every fused epilogue with partial tiles),
    vcl2 = L2-reduced virtual clusters wherever a split pays, novcl = hardware
    clusters only, push = hardware-cluster partials pushed to their owners by DSMEM bulk
    copies (instead of pulled after a cluster barrier), nochain = separate GEMM launches
    instead of the persistent per-layer GEMM chain kernels (the decode default, bf16 and
    QSUN), l2chain = the chains over plain CTAs with every split phase reduced through L2
    (instead of 4-CTA clusters reducing over DSMEM), nogemv = QSUN decode batches of <= 16
    rows on the tcgen05 W4 GEMM instead of the small-batch W4 GEMV, gvchain = the small-batch
    W4 GEMV as a persistent layer chain (opt-in), tileready = the bf16 chain's activation
    loads waiting for the producing tiles instead of the whole previous phase (opt-in), gvcluster =
    the W4 GEMV's split tiles reduced over DSMEM in hardware clusters instead of through L2,
    gvbal0 / gvbal2 = the W4 GEMV without its balanced schedule (whole tiles + remainder
    spread contiguously) / with it also in place of the per-tile split, attntile = the decode
    attention starting on its QKV tiles as the previous layer chain publishes them (opt-in)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ)
    if sched == "vcl2":
        env["SUN_GEMM_VCLUSTER"] = "2"
    elif sched == "novcl":
        env["SUN_GEMM_VCLUSTER"] = "0"
    elif sched == "push":
        env["SUN_GEMM_PUSH"] = "1"
    elif sched == "nochain":
        env["SUN_GEMM_CHAIN"] = "0"
    elif sched == "l2chain":
        env["SUN_CHAIN_CLUSTER"] = "0"
    elif sched == "nogemv":
        env["SUN_W4_GEMV"] = "0"
    elif sched == "gvchain":
        env["SUN_W4_GEMV_CHAIN"] = "1"
    elif sched == "tileready":
        env["SUN_CHAIN_TILE_READY"] = "1"
    elif sched == "gvcluster":
        env["SUN_GV_CLUSTER"] = "1"
    elif sched == "attntile":
        env["SUN_ATTN_TILE_READY"] = "1"
    elif sched in ("gvbal0", "gvbal2"):
        env["SUN_GV_BALANCE"] = sched[-1]
    else:
        env["SUN_GEMM_SCHED"] = sched
    sel = "(gemm or tiny or gemv) and not subprocess" if sched.startswith("gv") else "(gemm or tiny) and not subprocess"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        os.path.join(here, "test_kernels_gpu.py"), os.path.join(here, "test_decode_parity_gpu.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def _attn_ref(q, pool, layer, positions, bt, G):
    B, nq, d = q.shape
    out = torch.empty(B, nq * d, dtype=torch.float32)
    for b in range(B):
        ctx = int(positions[b]) + 1
        pages = bt[b, : (ctx + 15) // 16].tolist()
        kv = pool[pages, layer].float()  # [np, 2, nkv, 16, d]
        K = kv[:, 0].permute(1, 0, 2, 3).reshape(kv.shape[2], -1, d)[:, :ctx]
        V = kv[:, 1].permute(1, 0, 2, 3).reshape(kv.shape[2], -1, d)[:, :ctx]
        for h in range(nq):
            s = (K[h // G] @ q[b, h].float()) / math.sqrt(d)
            p = torch.softmax(s, dim=0)
            out[b, h * d:(h + 1) * d] = p @ V[h // G]
    return out


@pytest.mark.parametrize("d,nq,nkv", [(64, 8, 2), (128, 32, 8), (128, 40, 8)])
@pytest.mark.parametrize("pps", [0, 1, 3])
def test_attention_decode_matches_fp32(cuda, d, nq, nkv, pps):
    from paper_2603_02599_b200 import _lib, kernels

    L, num_pages, max_ctx = 2, 96, 600
    ctxs = [1, 15, 16, 17, 300, 599]
    B = len(ctxs)
    g = torch.Generator(device="cpu").manual_seed(d + nq + pps)
    pool = torch.randn(num_pages, L, 2, nkv, 16, d, generator=g).to(torch.bfloat16)
    perm = torch.randperm(num_pages, generator=g)
    maxp = (max_ctx + 15) // 16
    bt = torch.zeros(B, maxp, dtype=torch.int32)
    used = 0
    for b, c in enumerate(ctxs):
        n = (c + 15) // 16
        bt[b, :n] = perm[used:used + n].to(torch.int32)
        used += n
    positions = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32)
    q = torch.randn(B, nq, d, generator=g).to(torch.bfloat16)
    dims = _lib.SunDecoderDims(vocab=16, hidden=256, n_layers=L, n_q_heads=nq, n_kv_heads=nkv, head_dim=d,
                               ffn=256, page_size=16, max_context=max_ctx, weight_bits=16, group_size=128,
                               qkv_bias=0, rms_eps=1e-5)
    for layer in range(L):
        out = kernels.attention_decode(dims, pool.to(cuda), layer, q.to(cuda), positions.to(cuda), bt.to(cuda),
                                       pages_per_split=pps)
        ref = _attn_ref(q, pool, layer, positions, bt, nq // nkv)
        # P kept as bf16 hi+lo pair; output rounded to bf16 (1 ulp = 2^-8 relative)
        torch.testing.assert_close(out.float().cpu(), ref, rtol=1e-2, atol=2e-3)


@pytest.mark.parametrize("d,nq,nkv", [(64, 32, 8), (128, 32, 8), (128, 40, 8)])
@pytest.mark.parametrize("pps", [0, 8, 37, 1024])
def test_attention_decode_long_context(cuda, d, nq, nkv, pps):
    """Contexts of the BASELINE configs (C4 ~4k, C5 ~16k) with many splits: pps 8 gives
    up to 128 splits of one sequence merged by the split combine (online-softmax LSE
    merge over 1,000+ pages), 37 an odd split boundary, 1024 one split."""
    from paper_2603_02599_b200 import _lib, kernels

    L, max_ctx = 1, 16400
    ctxs = [16384, 4096, 4095, 9001, 16383, 1, 2049]
    B = len(ctxs)
    maxp = (max_ctx + 15) // 16
    num_pages = sum((c + 15) // 16 for c in ctxs) + 4
    g = torch.Generator(device="cpu").manual_seed(d * 3 + nq + pps)
    pool = (torch.randn(num_pages, L, 2, nkv, 16, d, generator=g) * 1.5).to(torch.bfloat16)
    perm = torch.randperm(num_pages, generator=g)
    bt = torch.zeros(B, maxp, dtype=torch.int32)
    used = 0
    for b, c in enumerate(ctxs):
        n = (c + 15) // 16
        bt[b, :n] = perm[used:used + n].to(torch.int32)
        used += n
    positions = torch.tensor([c - 1 for c in ctxs], dtype=torch.int32)
    q = (torch.randn(B, nq, d, generator=g) * 1.5).to(torch.bfloat16)
    dims = _lib.SunDecoderDims(vocab=16, hidden=256, n_layers=L, n_q_heads=nq, n_kv_heads=nkv, head_dim=d,
                               ffn=256, page_size=16, max_context=max_ctx, weight_bits=16, group_size=128,
                               qkv_bias=0, rms_eps=1e-5)
    out = kernels.attention_decode(dims, pool.to(cuda), 0, q.to(cuda), positions.to(cuda), bt.to(cuda),
                                   pages_per_split=pps)
    ref = _attn_ref(q, pool, 0, positions, bt, nq // nkv)
    torch.testing.assert_close(out.float().cpu(), ref, rtol=1e-2, atol=2e-3)


def test_rmsnorm_matches_fp32(cuda):
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(7, 4096, generator=g)
    w = (1 + 0.1 * torch.randn(4096, generator=g)).to(torch.bfloat16)
    y = kernels.rmsnorm(x.to(cuda), w.to(cuda), 1e-5).cpu()
    ref = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    torch.testing.assert_close(y.float(), ref, rtol=8e-3, atol=1e-2)


@pytest.mark.parametrize("rows,k", [(256, 256), (300, 512), (4096, 4096)])
def test_w4_quantizer_bit_exact_vs_oracle(cuda, rows, k):
    """GPU quantiser == oracle restatement of SUN-W4, byte for byte (valid rows)."""
    import numpy as np

    from oracle import quant_ref
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(rows + k)
    w = (torch.randn(rows, k, generator=g) * 0.02).to(torch.bfloat16)
    w[0, :128] = 0  # all-zero group -> scale 0, q 0
    packed, scales = kernels.quantize_w4(w.to(cuda))
    q, s = quant_ref.quantize(w)
    p_ref, s_ref = quant_ref.pack(q, s)
    rows_pad = (rows + 127) // 128 * 128
    def by_row(p):  # SUN-W4 block [chunk 4][row 128][16 B] -> [rows_pad][k/2]
        return p.reshape(rows_pad // 128, k // 128, 4, 128, 16).transpose(0, 3, 1, 2, 4).reshape(rows_pad, -1)

    pg, pr = by_row(packed.cpu().numpy()), by_row(p_ref)
    assert np.array_equal(pg[:rows], pr[:rows])
    sg = scales.cpu().view(torch.int16).numpy().astype(np.uint16)  # [rows_pad/128, K/128, 128]
    by_row_s = lambda a: a[..., quant_ref.SCALE_POS].transpose(0, 2, 1).reshape(rows_pad, -1)  # noqa: E731
    assert np.array_equal(by_row_s(sg)[:rows], by_row_s(s_ref)[:rows])
    assert torch.equal(quant_ref.unpack(packed.cpu().numpy(), rows, k), q)


@pytest.mark.parametrize("n_out,k,batch", [(256, 256, 1), (768, 512, 8), (4096, 4096, 64), (1536, 14336, 128),
                                           (28672, 4096, 128), (512, 128, 256)])
def test_gemm_w4_matches_dequantized_fp32(cuda, n_out, k, batch):
    from oracle import quant_ref
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(n_out + k + batch)
    w = (torch.randn(n_out, k, generator=g) * 0.02).to(torch.bfloat16)
    x = torch.randn(_r16(batch), k, generator=g).to(torch.bfloat16)
    packed, scales = kernels.quantize_w4(w.to(cuda))
    out = kernels.gemm_w4(packed, scales, n_out, k, x.to(cuda), batch).cpu()
    q, s = quant_ref.quantize(w)
    deq = quant_ref.dequantize(q, s)  # bf16(q * s): the exact tcgen05 operand
    ref = x[:batch].float() @ deq.float().t()
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-4 * math.sqrt(k))


@pytest.mark.parametrize("n_out,k,batch", [(256, 256, 1), (300, 512, 5), (768, 512, 8), (4096, 4096, 9),
                                           (6144, 4096, 16), (28672, 4096, 16), (4096, 14336, 1), (1536, 14336, 3),
                                           (128, 128, 2), (24576, 4096, 4)])
def test_gemv_w4_matches_group_scaled_fp64(cuda, n_out, k, batch):
    """Small-batch W4 GEMV (stream-K, L2 partials): exactly sum_g s_g * sum_k q x up to
    fp32 summation order; and within the bf16 rounding of q*s of the tcgen05 operand."""
    from oracle import quant_ref
    from paper_2603_02599_b200 import kernels

    g = torch.Generator(device="cpu").manual_seed(n_out * 3 + k + batch)
    w = (torch.randn(n_out, k, generator=g) * 0.02).to(torch.bfloat16)
    x = torch.randn(_r16(batch), k, generator=g).to(torch.bfloat16)
    x[batch:] = float("nan")  # padding rows of the activation must not leak
    packed, scales = kernels.quantize_w4(w.to(cuda))
    ws = kernels.gemm_workspace(n_out, k, batch, cuda)
    out = kernels.gemm_w4(packed, scales, n_out, k, x.to(cuda), batch, workspace=ws, gemv=True)
    out2 = kernels.gemm_w4(packed, scales, n_out, k, x.to(cuda), batch, workspace=ws, gemv=True)
    acc = kernels.gemm_w4(packed, scales, n_out, k, x.to(cuda), batch, out=out.clone(), accumulate=True,
                          workspace=ws, gemv=True)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)  # deterministic stream-K reduction, self-resetting counters
    q, s = quant_ref.quantize(w)
    xs = x[:batch].double().view(batch, k // 128, 128)
    qs = q.double().view(n_out, k // 128, 128)
    exact = torch.einsum("bgk,ngk,ng->bn", xs, qs, s.double())
    torch.testing.assert_close(out.cpu().double(), exact, rtol=1e-4, atol=1e-4 * math.sqrt(k))
    torch.testing.assert_close(acc.cpu().double(), 2 * exact, rtol=1e-4, atol=2e-4 * math.sqrt(k))
    deq_ref = x[:batch].float() @ quant_ref.dequantize(q, s).float().t()
    torch.testing.assert_close(out.cpu(), deq_ref, rtol=1e-2, atol=2e-3 * math.sqrt(k) * 0.02 * 8)
