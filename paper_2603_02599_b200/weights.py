"""Random-init decoder weights (synthetic; no checkpoints offline) and their
B200 device layout.

``init_weights`` returns the standard layout (HF-like names, one tensor per
projection) that the oracle also consumes; ``DeviceWeights`` re-lays it out for
the kernels (fused QKV rows, 64-row interleaved gate/up blocks, optional QSUN
W4 packing done by the GPU quantiser) and exposes the C ``SunWeights`` struct.
Task-specific prefill modules θ_p^τ are seeded perturbations of the frozen
decode module θ_d (θ_d frozen, θ_p^τ tuned per task).
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .spec import DecoderSpec

BF16 = torch.bfloat16


def _randn(shape, gen, device, std):
    return (torch.randn(*shape, generator=gen, device=device, dtype=torch.float32) * std).to(BF16)


def init_weights(spec: DecoderSpec, seed: int = 0, device: str | torch.device = "cpu") -> dict:
    """θ_d ~ N(0, init_std) for every matrix, RMSNorm gains 1 + N(0, 0.02)."""
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(seed)
    h, d = spec.hidden, spec.head_dim
    qd, kd = spec.n_q_heads * d, spec.n_kv_heads * d
    s = spec.init_std
    es = spec.embed_std if spec.embed_std is not None else s
    w = {"embed": _randn((spec.vocab, h), g, dev, es)}
    for l in range(spec.n_layers):
        w[f"l{l}.attn_norm"] = (1 + _randn((h,), g, dev, 0.02).float()).to(BF16)
        w[f"l{l}.wq"] = _randn((qd, h), g, dev, s)
        w[f"l{l}.wk"] = _randn((kd, h), g, dev, s)
        w[f"l{l}.wv"] = _randn((kd, h), g, dev, s)
        if spec.qkv_bias:
            w[f"l{l}.bq"] = _randn((qd,), g, dev, s)
            w[f"l{l}.bk"] = _randn((kd,), g, dev, s)
            w[f"l{l}.bv"] = _randn((kd,), g, dev, s)
        w[f"l{l}.wo"] = _randn((h, qd), g, dev, s)
        w[f"l{l}.ffn_norm"] = (1 + _randn((h,), g, dev, 0.02).float()).to(BF16)
        w[f"l{l}.wg"] = _randn((spec.ffn, h), g, dev, s)
        w[f"l{l}.wu"] = _randn((spec.ffn, h), g, dev, s)
        w[f"l{l}.wd"] = _randn((h, spec.ffn), g, dev, s)
    w["final_norm"] = torch.ones(h, dtype=BF16, device=dev)
    w["lm_head"] = w["embed"] if spec.tie_embeddings else _randn((spec.vocab, h), g, dev, spec.lm_head_std)
    if spec.greedy_margin > 0:
        if spec.tie_embeddings:
            raise ValueError("greedy_margin needs an untied lm_head")
        gp = torch.Generator(device=dev).manual_seed(seed * 7919 + 17)
        perm = torch.randperm(spec.vocab, generator=gp, device=dev)
        c = spec.greedy_margin / (h * es)
        for i in range(0, spec.vocab, 8192):  # chunked: bounded fp32 temporaries at V ~ 150k
            j = min(i + 8192, spec.vocab)
            w["lm_head"][i:j] = (w["lm_head"][i:j].float() + c * w["embed"][perm[i:j]].float()).to(BF16)
    return w


def perturb(spec: DecoderSpec, base: dict, seed: int, rel: float = 0.25) -> dict:
    """Task-specific prefill module θ_p^τ: every layer matrix of θ_d plus
    rel * init_std * N(0,1) noise (embedding, norms and lm_head shared)."""
    out = dict(base)
    dev = base["embed"].device
    g = torch.Generator(device=dev).manual_seed(1_000_003 * (seed + 1))
    for k, v in base.items():
        if k.startswith("l") and ".w" in k:
            out[k] = (v.float() + rel * spec.init_std * torch.randn(v.shape, generator=g, device=dev)).to(BF16)
    return out


def rope_tables(max_pos: int, head_dim: int, theta: float) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [max_pos, head_dim/2] fp32 of pos * theta^(-2i/d) (float64 math)."""
    half = head_dim // 2
    inv = theta ** (-(torch.arange(half, dtype=torch.float64) * 2.0) / head_dim)
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def interleave_gate_up(wg: torch.Tensor, wu: torch.Tensor) -> torch.Tensor:
    """[f,h] x2 -> [ceil(f/64)*128, h]: row 2i of block j = gate row 64j+i, row 2i+1 the
    matching up row (zero pad) — the SWIGLU epilogue pairs them with one lane shuffle."""
    f, h = wg.shape
    nb = (f + 63) // 64
    pad = nb * 64 - f
    gp = torch.cat([wg, wg.new_zeros(pad, h)]) if pad else wg
    up = torch.cat([wu, wu.new_zeros(pad, h)]) if pad else wu
    return torch.stack([gp.view(nb, 64, h), up.view(nb, 64, h)], dim=2).reshape(nb * 128, h)


class DeviceWeights:
    """The frozen module's tensors in the kernels' layout on one GPU."""

    def __init__(self, spec: DecoderSpec, w: dict, device: torch.device, max_context: int,
                 free_source: bool = False):
        from . import kernels

        self.spec = spec
        dev = torch.device(device)
        self.device = dev
        to = lambda t: t.to(dev, non_blocking=True).contiguous()  # noqa: E731
        self.embed = to(w["embed"])
        self.final_norm = to(w["final_norm"])
        # lm_head stays bf16, stored SUN-BLK for the GEMM stream
        self.lm_head = kernels.block_weights(self.embed if spec.tie_embeddings else to(w["lm_head"]))
        if free_source and not spec.tie_embeddings:
            w.pop("lm_head", None)
        cos, sin = rope_tables(max_context, spec.head_dim, spec.rope_theta)
        self.rope_cos, self.rope_sin = cos.to(dev), sin.to(dev)
        self.layers = []
        for l in range(spec.n_layers):
            L = {"attn_norm": to(w[f"l{l}.attn_norm"]), "ffn_norm": to(w[f"l{l}.ffn_norm"])}
            qkv = torch.cat([to(w[f"l{l}.wq"]), to(w[f"l{l}.wk"]), to(w[f"l{l}.wv"])])
            gu = interleave_gate_up(to(w[f"l{l}.wg"]), to(w[f"l{l}.wu"]))
            mats = {"qkv": qkv, "o": to(w[f"l{l}.wo"]), "gate_up": gu, "down": to(w[f"l{l}.wd"])}
            del qkv, gu
            if spec.qkv_bias:
                L["b_qkv"] = torch.cat([to(w[f"l{l}.bq"]), to(w[f"l{l}.bk"]), to(w[f"l{l}.bv"])])
            for name, m in mats.items():
                if spec.weight_bits == 4:
                    L["w_" + name], L["s_" + name] = kernels.quantize_w4(m, spec.group_size)
                else:
                    L["w_" + name] = kernels.block_weights(m)
                del m
            if free_source:
                for k in ("wq", "wk", "wv", "wo", "wg", "wu", "wd"):
                    w.pop(f"l{l}.{k}", None)
            self.layers.append(L)
        self._build_struct()

    @classmethod
    def from_layout(cls, spec: DecoderSpec, embed: torch.Tensor, final_norm: torch.Tensor, lm_head: torch.Tensor,
                    layers: list[dict], device: torch.device, max_context: int) -> "DeviceWeights":
        """Tensors already in the kernels' layout (a checkpoint, checkpoint.py): nothing
        is quantised or re-blocked; only the RoPE tables are computed for max_context."""
        self = cls.__new__(cls)
        self.spec, self.device = spec, torch.device(device)
        need = ["attn_norm", "ffn_norm", "w_qkv", "w_o", "w_gate_up", "w_down"]
        if spec.weight_bits == 4:
            need += ["s_qkv", "s_o", "s_gate_up", "s_down"]
        if spec.qkv_bias:
            need.append("b_qkv")
        for l, L in enumerate(layers):
            missing = [k for k in need if k not in L]
            if missing:
                raise ValueError(f"layer {l}: missing {missing}")
        if len(layers) != spec.n_layers:
            raise ValueError(f"{len(layers)} layers for a {spec.n_layers}-layer spec")
        self.embed, self.final_norm, self.lm_head, self.layers = embed, final_norm, lm_head, layers
        cos, sin = rope_tables(max_context, spec.head_dim, spec.rope_theta)
        self.rope_cos, self.rope_sin = cos.to(self.device), sin.to(self.device)
        self._build_struct()
        return self

    def _build_struct(self) -> None:
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        arr = (_lib.SunLayerWeights * len(self.layers))()
        for i, L in enumerate(self.layers):
            arr[i] = _lib.SunLayerWeights(
                ptr(L["attn_norm"]), ptr(L["w_qkv"]), ptr(L.get("s_qkv")), ptr(L.get("b_qkv")),
                ptr(L["w_o"]), ptr(L.get("s_o")), ptr(L["ffn_norm"]), ptr(L["w_gate_up"]), ptr(L.get("s_gate_up")),
                ptr(L["w_down"]), ptr(L.get("s_down")))
        self._layer_arr = arr
        self.struct = _lib.SunWeights(self.embed.data_ptr(), self.final_norm.data_ptr(), self.lm_head.data_ptr(),
                                      self.rope_cos.data_ptr(), self.rope_sin.data_ptr(),
                                      ctypes.cast(arr, ctypes.POINTER(_lib.SunLayerWeights)))

    def nbytes(self) -> int:
        n = sum(t.numel() * t.element_size() for L in self.layers for t in L.values())
        return n + self.embed.numel() * 2 + self.final_norm.numel() * 2 + self.lm_head.numel()


def std_layout_to_cpu(w: dict) -> dict:
    return {k: v.detach().cpu() for k, v in w.items()}


def logit_scale_note(spec: DecoderSpec) -> float:
    """Expected logit std for unit-RMS normalised inputs (margin sanity)."""
    return spec.lm_head_std * math.sqrt(spec.hidden)
