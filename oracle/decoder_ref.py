"""ORACLE — test infrastructure only. CPU fp32 restatement of the SUN decoder.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU baseline,
never as a product code path.

What it restates
----------------
The reference (poolsim) has no decoder arithmetic: the decode step exists only
as the price ``D + (W + sum KV)/(mbu*BW)`` (pkg/src/poolsim/costmodel.py:101-113)
and the prefill/decode split only as per-phase weight bits
(pkg/src/poolsim/domain.py:116-133). The math is defined by the paper:

* PAPER.md:165-168 (Eq. 2): prefill module P_θp(X) -> (p(y1|X), C_X);
* PAPER.md:166-172 (Eq. 3): decode module D_θd(y_{t-1}, C_{<t-1}) -> (p(y_t|...), C_t);
* PAPER.md:176-184 (Eq. 4): C_{<=t} = C_X || C_{y<=t} — the decode module appends to
  the cache the task-specific prefill module produced;
* θ_d frozen and shared, θ_p^τ per task;
* QSUN = W4 symmetric group-128 weight-only, lm_head full precision
  (see quant_ref.py).

The block is a standard Llama-3 / Qwen2.5 decoder layer (pre-RMSNorm, GQA with
NeoX-style RoPE on q and k, SwiGLU MLP, optional QKV bias, untied or tied lm_head).

Parity status: **parity unpinned** for logits / greedy tokens / QSUN numerics —
no reference code computes them and the paper's stack (vLLM, LLM Compressor AWQ)
is neither vendored nor pinned. The rounding points below are the
ones the B200 path uses, so the comparison isolates accumulation-order effects:

  resid fp32;  RMSNorm is factored: xg = bf16(resid * g), r = rsqrt(mean(resid^2)+eps),
  and a normed projection is (xg @ W^T) * r  (= W.(x*r*g); the B200 GEMMs apply r
  per batch column in their epilogues, so no separate norm kernel exists)
  q,k = bf16(rope((xg @ Wqkv^T) * r + b)),  v = bf16(...)     (K cached post-RoPE)
  attn = bf16(softmax(q k^T / sqrt(d)) v)                     (fp32 softmax)
  resid += attn @ Wo^T;  act = bf16(silu(g) * u) with g,u = (xg @ W^T) * r
  resid += act @ Wdown^T
  logits = fp32((bf16(resid * g_final) @ lm_head^T) * r);  next = argmax (lowest index on ties)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

BF16 = torch.bfloat16


@dataclass(frozen=True)
class OracleSpec:
    vocab: int
    hidden: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool = False


def bf(x: torch.Tensor) -> torch.Tensor:
    """Round fp32 -> bf16 -> fp32 (round-to-nearest-even), the GPU's storage rounding."""
    return x.to(BF16).float()


def rope_tables(max_pos: int, head_dim: int, theta: float) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [max_pos, head_dim/2] fp32 of angle pos * theta^(-2i/d), computed in float64."""
    half = head_dim // 2
    inv = theta ** (-(torch.arange(half, dtype=torch.float64) * 2.0) / head_dim)
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def rmsnorm(x: torch.Tensor, g: torch.Tensor, eps: float, rnd=None) -> torch.Tensor:
    r = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
    return (rnd or bf)(x * r * g.float())


def norm_factored(x: torch.Tensor, g: torch.Tensor, eps: float, rnd=None) -> tuple[torch.Tensor, torch.Tensor]:
    """(xg, r): xg = round(x * g), r = rsqrt(mean(x^2) + eps) per row; rmsnorm = xg * r."""
    r = torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)
    return (rnd or bf)(x * g.float()), r


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [..., d] fp32, cos/sin [..., d/2] broadcastable; NeoX rotate-half."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def argmax_lowest(logits: torch.Tensor) -> torch.Tensor:
    m = logits.max(dim=-1, keepdim=True).values
    idx = torch.arange(logits.shape[-1], device=logits.device).expand_as(logits)
    return torch.where(logits == m, idx, torch.full_like(idx, logits.shape[-1])).min(dim=-1).values


class OracleDecoder:
    """Weights: dict of CPU bf16 tensors in the standard (HF-like) layout:
    embed [V,h], final_norm [h], lm_head [V,h], and per layer l:
    attn_norm, wq [nq*d,h], wk [nkv*d,h], wv [nkv*d,h], (bq, bk, bv), wo [h,nq*d],
    ffn_norm, wg [f,h], wu [f,h], wd [h,f].
    """

    def __init__(self, spec: OracleSpec, weights: dict, max_pos: int, round_bf16: bool = True,
                 device: str | torch.device = "cpu"):
        """round_bf16=False drops every bf16 storage rounding (pure fp32 model), the
        mode used to pin the block definition against transformers' Llama / Qwen2.

        device: where the same fp32 arithmetic runs. "cpu" is the oracle proper;
        the BASELINE-shape parity tests (contexts up to 16k, ~1e14 flop of prefill)
        run these very torch ops on a CUDA device with TF32 disabled (fp32 cuBLAS /
        elementwise, nothing from libsun_b200.so), pinned equal to the CPU run by
        tests/test_oracle_device_gpu.py."""
        self.s = spec
        self.dev = torch.device(device)
        if self.dev.type == "cuda":
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
        self.w = {k: (v.to(self.dev).float() if torch.is_tensor(v) else v) for k, v in weights.items()}
        cos, sin = rope_tables(max_pos, spec.head_dim, spec.rope_theta)
        self.cos, self.sin = cos.to(self.dev), sin.to(self.dev)
        self.rnd = bf if round_bf16 else (lambda x: x)

    # -- one layer over T new positions of one sequence ------------------------------
    def _layer(self, l: int, resid: torch.Tensor, pos: torch.Tensor, kcache: list, vcache: list):
        s, w = self.s, self.w
        d, nq, nkv = s.head_dim, s.n_q_heads, s.n_kv_heads
        T = resid.shape[0]
        xg, r = norm_factored(resid, w[f"l{l}.attn_norm"], s.rms_eps, self.rnd)
        q = (xg @ w[f"l{l}.wq"].t()) * r
        k = (xg @ w[f"l{l}.wk"].t()) * r
        v = (xg @ w[f"l{l}.wv"].t()) * r
        if s.qkv_bias:
            q = q + w[f"l{l}.bq"]
            k = k + w[f"l{l}.bk"]
            v = v + w[f"l{l}.bv"]
        cs, sn = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        q = self.rnd(rope(q.view(T, nq, d), cs, sn))
        k = self.rnd(rope(k.view(T, nkv, d), cs, sn))
        v = self.rnd(v.view(T, nkv, d))
        K = torch.cat([kcache[l], k], 0) if kcache[l] is not None else k
        V = torch.cat([vcache[l], v], 0) if vcache[l] is not None else v
        kcache[l], vcache[l] = K, V
        G = nq // nkv
        n_past = K.shape[0] - T
        out = torch.empty(T, nq, d, device=self.dev)
        causal = (torch.arange(K.shape[0], device=self.dev)[None, :] >
                  (n_past + torch.arange(T, device=self.dev))[:, None]) if T > 1 else None
        for h in range(nq):
            sc = (q[:, h, :] @ K[:, h // G, :].t()) / math.sqrt(d)  # [T, ctx]
            if causal is not None:
                sc = sc.masked_fill(causal, float("-inf"))
            out[:, h, :] = torch.softmax(sc, dim=-1) @ V[:, h // G, :]
        attn = self.rnd(out.reshape(T, nq * d))
        resid = resid + attn @ w[f"l{l}.wo"].t()
        xg, r = norm_factored(resid, w[f"l{l}.ffn_norm"], s.rms_eps, self.rnd)
        g = (xg @ w[f"l{l}.wg"].t()) * r
        u = (xg @ w[f"l{l}.wu"].t()) * r
        act = self.rnd(g / (1.0 + torch.exp(-g)) * u)
        return resid + act @ w[f"l{l}.wd"].t()

    def forward(self, tokens: list[int], start: int, cache: dict | None):
        """Run positions start..start+len(tokens)-1 of one sequence.

        Returns (logits of the last position [V] fp32, cache) where cache holds
        per-layer K/V [ctx, nkv, d] (bf16-valued fp32).
        """
        s, w = self.s, self.w
        if cache is None:
            cache = {"k": [None] * s.n_layers, "v": [None] * s.n_layers}
        pos = torch.arange(start, start + len(tokens), device=self.dev)
        resid = w["embed"][torch.tensor(tokens, device=self.dev)].clone()
        for l in range(s.n_layers):
            resid = self._layer(l, resid, pos, cache["k"], cache["v"])
        xg, r = norm_factored(resid[-1:], w["final_norm"], s.rms_eps, self.rnd)
        logits = ((xg @ w["lm_head"].t()) * r)[0]
        return logits, cache

    # Eq. 2: prefill module P_θp(X) -> (first-token logits, C_X)
    def prefill(self, prompt: list[int]):
        return self.forward(prompt, 0, None)

    # Eq. 3: decode module D_θd(y_{t-1}, C_{<t-1}) -> (logits, C_t)
    def decode(self, token: int, pos: int, cache: dict):
        return self.forward([token], pos, cache)


def greedy_shared_decode(prefills: list[OracleDecoder], decoder: OracleDecoder, prompts: list[list[int]],
                         module_of: list[int], n_steps: int):
    """Reference semantics of SUN: request i is prefilled by
    its task module prefills[module_of[i]], then decoded greedily by the one shared
    decoder. Returns (tokens [B][1+n_steps], per-step logits [n_steps][B][V],
    per-step top-2 margins)."""
    toks, caches, logs, margins = [], [], [], []
    for p, m in zip(prompts, module_of):
        lg, c = prefills[m].prefill(p)
        toks.append([int(argmax_lowest(lg[None])[0])])
        caches.append(c)
    for t in range(n_steps):
        step_logits = []
        for i, p in enumerate(prompts):
            lg, caches[i] = decoder.decode(toks[i][-1], len(p) + t, caches[i])
            step_logits.append(lg)
            toks[i].append(int(argmax_lowest(lg[None])[0]))
        L = torch.stack(step_logits)
        top2 = L.topk(2, dim=-1).values
        margins.append((top2[:, 0] - top2[:, 1]))
        logs.append(L)
    return toks, logs, margins


def teacher_forced(prefills: list[OracleDecoder], decoder: OracleDecoder, prompts: list[list[int]],
                   module_of: list[int], tokens: list[list[int]]):
    """Score a given token history (e.g. the GPU's greedy output) with the oracle:
    returns per-sequence logits [1 + n_steps, V] where row 0 is the prefill
    module's first-token distribution and row t+1 the decoder's after consuming
    tokens[i][t] at position len(prompt) + t."""
    out = []
    for i, (p, m) in enumerate(zip(prompts, module_of)):
        lg, c = prefills[m].prefill(p)
        rows = [lg]
        for t, tok in enumerate(tokens[i][:-1]):
            lg, c = decoder.decode(tok, len(p) + t, c)
            rows.append(lg)
        out.append(torch.stack(rows))
    return out


def decode_batch_layers(dec: OracleDecoder, tokens: list[int], positions: list[int], caches: list[dict],
                        layers: range, lm_head: bool = True):
    """Batched CPU decode step (the timed CPU baseline): the linear layers run on
    the whole [B, h] batch (weights streamed once per step, like the GPU path),
    attention per sequence over its own cache. ``layers`` may be a subset (the
    bench's bounded sample); caches hold K/V [ctx, nkv, d] per layer index.
    Returns logits [B, V] (or the residual stream if lm_head=False)."""
    s, w = dec.s, dec.w
    d, nq, nkv = s.head_dim, s.n_q_heads, s.n_kv_heads
    G = nq // nkv
    B = len(tokens)
    pos = torch.tensor(positions)
    resid = w["embed"][torch.tensor(tokens)].clone()
    for l in layers:
        xg, r = norm_factored(resid, w[f"l{l}.attn_norm"], s.rms_eps)
        q, k, v = (xg @ w[f"l{l}.wq"].t()) * r, (xg @ w[f"l{l}.wk"].t()) * r, (xg @ w[f"l{l}.wv"].t()) * r
        if s.qkv_bias:
            q, k, v = q + w[f"l{l}.bq"], k + w[f"l{l}.bk"], v + w[f"l{l}.bv"]
        cs, sn = dec.cos[pos][:, None, :], dec.sin[pos][:, None, :]
        q = bf(rope(q.view(B, nq, d), cs, sn))
        k = bf(rope(k.view(B, nkv, d), cs, sn))
        v = bf(v.view(B, nkv, d))
        out = torch.empty(B, nq, d)
        for b in range(B):
            K = torch.cat([caches[b]["k"][l], k[b:b + 1]])
            V = torch.cat([caches[b]["v"][l], v[b:b + 1]])
            caches[b]["k"][l], caches[b]["v"][l] = K, V
            qg = q[b].view(nkv, G, d)
            sc = torch.einsum("hgd,thd->hgt", qg, K) / math.sqrt(d)
            out[b] = torch.einsum("hgt,thd->hgd", torch.softmax(sc, -1), V).reshape(nq, d)
        attn = bf(out.reshape(B, nq * d))
        resid = resid + attn @ w[f"l{l}.wo"].t()
        xg, r = norm_factored(resid, w[f"l{l}.ffn_norm"], s.rms_eps)
        g, u = (xg @ w[f"l{l}.wg"].t()) * r, (xg @ w[f"l{l}.wu"].t()) * r
        resid = resid + bf(g / (1.0 + torch.exp(-g)) * u) @ w[f"l{l}.wd"].t()
    if not lm_head:
        return resid
    xg, r = norm_factored(resid, w["final_norm"], s.rms_eps)
    return (xg @ w["lm_head"].t()) * r
