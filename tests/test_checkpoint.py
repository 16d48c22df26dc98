"""QSUN checkpoints on CPU (no kernels): the SUNCKPT file round trip of a W4
module's device layout, and the compressed-tensors int4 packing rule
(paper_2603_02599_b200/checkpoint.py; QSUN's offline pipeline PAPER.md:515-519)."""
import numpy as np
import torch

from oracle import quant_ref
from paper_2603_02599_b200 import checkpoint
from dataclasses import replace

from paper_2603_02599_b200.spec import TINY
from paper_2603_02599_b200.weights import DeviceWeights, init_weights


def _cpu_w4_module(spec, seed=0):
    """A W4 DeviceWeights on CPU laid out by the oracle's SUN-W4 packer (test only)."""
    w = init_weights(spec, seed)
    layers = []
    for l in range(spec.n_layers):
        L = {"attn_norm": w[f"l{l}.attn_norm"], "ffn_norm": w[f"l{l}.ffn_norm"],
             "b_qkv": torch.cat([w[f"l{l}.bq"], w[f"l{l}.bk"], w[f"l{l}.bv"]])}
        mats = {"qkv": torch.cat([w[f"l{l}.wq"], w[f"l{l}.wk"], w[f"l{l}.wv"]]), "o": w[f"l{l}.wo"],
                "gate_up": torch.cat([w[f"l{l}.wg"], w[f"l{l}.wu"]]), "down": w[f"l{l}.wd"]}
        for name, m in mats.items():
            q, s = quant_ref.quantize(m)
            p, sc = quant_ref.pack(q, s)
            L["w_" + name] = torch.from_numpy(p.copy())
            L["s_" + name] = torch.from_numpy(sc.astype(np.int16)).view(torch.bfloat16)
        layers.append(L)
    lm = torch.randint(0, 256, (spec.vocab * spec.hidden * 2,), dtype=torch.uint8)  # opaque SUN-BLK bytes
    return DeviceWeights.from_layout(spec.with_bits(4), w["embed"], w["final_norm"], lm, layers, torch.device("cpu"),
                                     64)


def test_sunckpt_round_trip_bit_identical(tmp_path):
    dw = _cpu_w4_module(replace(TINY, name="tiny", ffn=768, qkv_bias=True))  # W4 needs K % 128 == 0
    path = tmp_path / "tiny_w4.sunckpt"
    checkpoint.save(path, dw)
    header, base = checkpoint.read_header(path)
    assert header["format"] == "sun-w4" and base % checkpoint.ALIGN == 0
    assert all(e["offset"] % checkpoint.ALIGN == 0 for e in header["tensors"])
    back = checkpoint.load(path, "cpu", 64)
    assert back.spec == dw.spec
    for (n1, a), (n2, b) in zip(checkpoint._named_tensors(dw), checkpoint._named_tensors(back)):
        assert n1 == n2 and a.dtype == b.dtype and a.shape == b.shape
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8)), n1
    assert back.nbytes() == dw.nbytes()


def test_sunckpt_rejects_foreign_files(tmp_path):
    p = tmp_path / "x.bin"
    p.write_bytes(b"not a checkpoint at all")
    import pytest

    with pytest.raises(ValueError):
        checkpoint.read_header(p)
    old = tmp_path / "v1.sunckpt"  # the previous layout (gate/up in 64-row blocks) is refused by version
    old.write_bytes(b"SUNCKPT\x01" + bytes(8))
    with pytest.raises(ValueError, match="version 1"):
        checkpoint.read_header(old)


def test_compressed_tensors_packing_rule():
    """Element 8j+i of a row sits in nibble i of int32 word j as q + 8 (two's complement view)."""
    g = torch.Generator().manual_seed(3)
    q = torch.randint(-8, 8, (5, 64), generator=g)
    words = checkpoint.pack_compressed_tensors(q)
    assert words.dtype == torch.int32 and words.shape == (5, 8)
    u = words.numpy().view(np.uint32)
    for r in range(5):
        for k in range(64):
            assert ((int(u[r, k // 8]) >> (4 * (k % 8))) & 0xF) - 8 == int(q[r, k])


def test_compressed_tensors_import_rejects_non_w4_layers():
    """A linear layer that is not pack-quantized int4 (missing weight_scale, or a
    weight_shape that disagrees with the packing) is refused before any device work."""
    import pytest

    from paper_2603_02599_b200.errors import UnsupportedShape

    spec = replace(TINY, name="tiny", ffn=768, n_layers=1)
    w = init_weights(spec, 0)
    q, s = quant_ref.quantize(w["l0.wq"])
    base = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
            "lm_head.weight": w["lm_head"], "model.layers.0.input_layernorm.weight": w["l0.attn_norm"],
            "model.layers.0.post_attention_layernorm.weight": w["l0.ffn_norm"],
            "model.layers.0.self_attn.q_proj.weight_packed": checkpoint.pack_compressed_tensors(q)}
    with pytest.raises(UnsupportedShape):  # no weight_scale
        checkpoint.from_compressed_tensors(spec, base, "cpu", 64)
    bad = dict(base)
    bad["model.layers.0.self_attn.q_proj.weight_scale"] = s
    bad["model.layers.0.self_attn.q_proj.weight_shape"] = torch.tensor([q.shape[0], q.shape[1] * 2])
    with pytest.raises(UnsupportedShape):  # weight_shape disagrees with the packed K
        checkpoint.from_compressed_tensors(spec, bad, "cpu", 64)
