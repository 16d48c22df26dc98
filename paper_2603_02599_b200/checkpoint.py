"""QSUN / SUN checkpoints: the frozen decode module θ_d stored in the kernels' own
device layout, and import of LLM-Compressor-style W4A16 checkpoints.

QSUN quantises the shared decoder once, offline (AWQ through
LLM Compressor, 4-bit symmetric, group 128, lm_head kept in bf16) and serves the
quantised checkpoint. Here that is two load paths that never re-quantise:

* ``save`` / ``load`` — a single-file ``SUNCKPT`` checkpoint of a ``DeviceWeights``:
  SUN-W4 packed blocks + tile-major scales (or SUN-BLK bf16 blocks), norms, biases,
  embedding and the SUN-BLK lm_head, byte for byte as they sit in HBM. Loading is
  one read per tensor and a host->device copy; the result is bit-identical to the
  module that was saved (tests/test_checkpoint*.py).
* ``from_compressed_tensors`` — a Hugging Face state dict in the compressed-tensors
  "pack-quantized" layout (``*.weight_packed`` int32 [rows, K/8], ``*.weight_scale``
  bf16 [rows, K/128], symmetric int4, group 128: what LLM Compressor writes for
  W4A16), re-laid out to SUN-W4 on the GPU by ``sun_import_w4_ct`` (nibble and
  block permutation only: the operand bf16(q * s) is the checkpoint's).
  compressed-tensors itself is not in this image; the layout is restated from its
  published packing rule (``pack_to_int32``: unsigned q + 8, element 8j+i of a row
  in bits 4i..4i+3 of word j), version unpinned.

File layout: b"SUNCKPT\\x02", u64 little-endian header length, UTF-8 JSON header
{"format", "spec", "tensors": [{"name", "dtype", "shape", "offset", "nbytes"}]},
then each tensor's raw bytes at its offset (4 KiB aligned).
"""
from __future__ import annotations

import dataclasses
import json
import os
import struct

import numpy as np
import torch

from .errors import UnsupportedShape
from .spec import DecoderSpec

MAGIC = b"SUNCKPT\x02"  # \x02: gate/up pair-interleaved rows (weights.interleave_gate_up)
ALIGN = 4096
_DT = {torch.uint8: "u8", torch.bfloat16: "bf16", torch.float32: "f32", torch.int32: "i32"}
_DT_INV = {v: k for k, v in _DT.items()}
_NP = {"u8": np.uint8, "bf16": np.uint16, "f32": np.float32, "i32": np.int32}
_LAYER_KEYS = ("attn_norm", "ffn_norm", "w_qkv", "s_qkv", "b_qkv", "w_o", "s_o", "w_gate_up", "s_gate_up",
               "w_down", "s_down")


def _named_tensors(dw) -> list[tuple[str, torch.Tensor]]:
    out = [("embed", dw.embed), ("final_norm", dw.final_norm), ("lm_head", dw.lm_head)]
    for l, L in enumerate(dw.layers):
        out += [(f"l{l}.{k}", L[k]) for k in _LAYER_KEYS if k in L]
    return out


def save(path: str | os.PathLike, dw) -> None:
    """Write ``DeviceWeights`` ``dw`` (bf16 or QSUN W4) as a SUNCKPT file."""
    entries, off = [], 0
    named = _named_tensors(dw)
    for name, t in named:
        nbytes = t.numel() * t.element_size()
        entries.append({"name": name, "dtype": _DT[t.dtype], "shape": list(t.shape), "offset": off, "nbytes": nbytes})
        off += (nbytes + ALIGN - 1) // ALIGN * ALIGN
    fmt = "sun-w4" if dw.spec.weight_bits == 4 else "sun-bf16"
    header = json.dumps({"format": fmt, "spec": dataclasses.asdict(dw.spec), "tensors": entries}).encode()
    base = (len(MAGIC) + 8 + len(header) + ALIGN - 1) // ALIGN * ALIGN
    tmp = f"{os.fspath(path)}.tmp"
    with open(tmp, "wb") as f:
        f.write(MAGIC + struct.pack("<Q", len(header)) + header)
        for (name, t), e in zip(named, entries):
            f.seek(base + e["offset"])
            f.write(t.detach().contiguous().view(torch.uint8).reshape(-1).cpu().numpy().tobytes())
        f.truncate(base + off)
    os.replace(tmp, path)


def read_header(path: str | os.PathLike) -> tuple[dict, int]:
    with open(path, "rb") as f:
        magic = f.read(len(MAGIC))
        if magic[:7] == MAGIC[:7] and magic != MAGIC:
            raise ValueError(f"{path}: SUNCKPT version {magic[7]} (this build reads {MAGIC[7]}): re-export it")
        if magic != MAGIC:
            raise ValueError(f"{path}: not a SUNCKPT checkpoint")
        (n,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(n))
    return header, (len(MAGIC) + 8 + n + ALIGN - 1) // ALIGN * ALIGN


def load(path: str | os.PathLike, device: str | torch.device, max_context: int):
    """SUNCKPT file -> ``DeviceWeights`` on ``device`` (no quantisation, no re-layout)."""
    from .weights import DeviceWeights

    header, base = read_header(path)
    spec = DecoderSpec(**header["spec"])
    want = "sun-w4" if spec.weight_bits == 4 else "sun-bf16"
    if header["format"] != want:
        raise ValueError(f"{path}: format {header['format']!r} does not match its spec ({want})")
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    dev = torch.device(device)
    tensors = {}
    for e in header["tensors"]:
        raw = mm[base + e["offset"]: base + e["offset"] + e["nbytes"]]
        host = torch.from_numpy(np.array(raw.view(_NP[e["dtype"]])))
        if e["dtype"] == "bf16":
            host = host.view(torch.bfloat16)
        tensors[e["name"]] = host.reshape(e["shape"]).to(dev)
    del mm
    layers = [{k: tensors[f"l{l}.{k}"] for k in _LAYER_KEYS if f"l{l}.{k}" in tensors} for l in range(spec.n_layers)]
    return DeviceWeights.from_layout(spec, tensors["embed"], tensors["final_norm"], tensors["lm_head"], layers, dev,
                                     max_context)


# --- compressed-tensors (LLM Compressor W4A16) import ---------------------------------

def _hf(l: int, mod: str) -> str:
    return f"model.layers.{l}.{mod}"


def from_compressed_tensors(spec: DecoderSpec, state: dict, device: str | torch.device, max_context: int):
    """HF state dict (Llama / Qwen2 names) with W4A16 pack-quantized linear layers ->
    ``DeviceWeights`` of ``spec.with_bits(4)``. Embedding, norms, biases and lm_head are
    taken as stored (bf16); every decoder linear layer must be pack-quantized int4."""
    from . import kernels
    from .weights import DeviceWeights, interleave_gate_up

    spec = spec if spec.weight_bits == 4 else spec.with_bits(4)
    if spec.group_size != 128:
        raise UnsupportedShape("SUN-W4 implements group size 128")
    dev = torch.device(device)
    to = lambda t: t.to(dev).contiguous()  # noqa: E731

    def q(name: str) -> tuple[torch.Tensor, torch.Tensor]:
        packed, scale = state.get(name + ".weight_packed"), state.get(name + ".weight_scale")
        if packed is None or scale is None:
            raise UnsupportedShape(f"{name}: not a pack-quantized W4 tensor (weight_packed / weight_scale)")
        shape = state.get(name + ".weight_shape")
        if shape is not None and int(shape[1]) != packed.shape[1] * 8:
            raise UnsupportedShape(f"{name}: weight_shape {list(map(int, shape))} vs packed {tuple(packed.shape)}")
        return to(packed), to(scale)

    layers = []
    for l in range(spec.n_layers):
        L = {"attn_norm": to(state[_hf(l, "input_layernorm.weight")]),
             "ffn_norm": to(state[_hf(l, "post_attention_layernorm.weight")])}
        parts = [q(_hf(l, f"self_attn.{p}_proj")) for p in ("q", "k", "v")]
        mats = {"qkv": (torch.cat([p for p, _ in parts]), torch.cat([s for _, s in parts])),
                "o": q(_hf(l, "self_attn.o_proj"))}
        (gp, gs), (up, us) = q(_hf(l, "mlp.gate_proj")), q(_hf(l, "mlp.up_proj"))
        mats["gate_up"] = (interleave_gate_up(gp, up), interleave_gate_up(gs, us))
        mats["down"] = q(_hf(l, "mlp.down_proj"))
        if spec.qkv_bias:
            L["b_qkv"] = torch.cat([to(state[_hf(l, f"self_attn.{p}_proj.bias")]) for p in ("q", "k", "v")])
        for name, (packed, scale) in mats.items():
            L["w_" + name], L["s_" + name] = kernels.import_w4_ct(packed, scale, spec.group_size)
        layers.append(L)
    embed = to(state["model.embed_tokens.weight"])
    lm = embed if spec.tie_embeddings else to(state["lm_head.weight"])
    return DeviceWeights.from_layout(spec, embed, to(state["model.norm.weight"]), kernels.block_weights(lm), layers,
                                     dev, max_context)


def pack_compressed_tensors(q: torch.Tensor) -> torch.Tensor:
    """int q in [-8, 7], [rows, K] -> compressed-tensors int32 [rows, K/8] (element 8j+i in
    nibble i of word j, offset-binary). The writer side of the import, for checkpoints made
    here and for tests."""
    rows, k = q.shape
    u = (q.to(torch.int64) + 8).view(rows, k // 8, 8)
    word = torch.zeros(rows, k // 8, dtype=torch.int64, device=q.device)
    for i in range(8):
        word |= u[..., i] << (4 * i)
    return (word - ((word >> 31) << 32)).to(torch.int32)  # two's complement view of the uint32
