"""QSUN checkpoint load paths on the B200 (checkpoint.py): a
compressed-tensors W4A16 state dict imported by sun_import_w4_ct, and a SUNCKPT
file saved and loaded back, both give a decode module bit-identical to the one
the GPU quantiser builds from the same bf16 weights — same bytes in HBM, same
decode logits — with no quantisation on either load path."""
from dataclasses import replace

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ct_state(spec, w):
    """HF-named compressed-tensors state dict of θ_d (oracle quantiser: test only)."""
    from oracle import quant_ref
    from paper_2603_02599_b200.checkpoint import pack_compressed_tensors

    st = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"], "lm_head.weight": w["lm_head"]}
    names = {"wq": "self_attn.q_proj", "wk": "self_attn.k_proj", "wv": "self_attn.v_proj", "wo": "self_attn.o_proj",
             "wg": "mlp.gate_proj", "wu": "mlp.up_proj", "wd": "mlp.down_proj"}
    for l in range(spec.n_layers):
        p = f"model.layers.{l}."
        st[p + "input_layernorm.weight"] = w[f"l{l}.attn_norm"]
        st[p + "post_attention_layernorm.weight"] = w[f"l{l}.ffn_norm"]
        for k, hf in names.items():
            q, s = quant_ref.quantize(w[f"l{l}.{k}"])
            st[p + hf + ".weight_packed"] = pack_compressed_tensors(q)
            st[p + hf + ".weight_scale"] = s
            st[p + hf + ".weight_shape"] = torch.tensor(list(q.shape))
        if spec.qkv_bias:
            for k, hf in (("bq", "q_proj"), ("bk", "k_proj"), ("bv", "v_proj")):
                st[p + f"self_attn.{hf}.bias"] = w[f"l{l}.{k}"]
    return st


@pytest.mark.parametrize("rows,k", [(256, 256), (300, 512), (4096, 4096)])
def test_import_w4_ct_equals_quantizer(cuda, rows, k):
    from oracle import quant_ref
    from paper_2603_02599_b200 import kernels
    from paper_2603_02599_b200.checkpoint import pack_compressed_tensors

    g = torch.Generator(device="cpu").manual_seed(rows * 3 + k)
    w = (torch.randn(rows, k, generator=g) * 0.02).to(torch.bfloat16)
    w[1, 128:256] = 0
    q, s = quant_ref.quantize(w)
    p_imp, s_imp = kernels.import_w4_ct(pack_compressed_tensors(q).to(cuda), s.to(cuda))
    p_q, s_q = kernels.quantize_w4(w.to(cuda))
    torch.cuda.synchronize()
    assert torch.equal(p_imp, p_q) and torch.equal(s_imp.view(torch.int16), s_q.view(torch.int16))
    p_ref, _ = quant_ref.pack(q, s)
    rows_pad = (rows + 127) // 128 * 128
    by_row = lambda p: p.reshape(rows_pad // 128, k // 128, 4, 128, 16).transpose(0, 3, 1, 2, 4).reshape(rows_pad, -1)
    assert np.array_equal(by_row(p_imp.cpu().numpy())[:rows], by_row(p_ref)[:rows])


def _decode_logits(spec, dw, cuda, steps=3):
    from paper_2603_02599_b200.kvpool import KvPool, pages_for
    from paper_2603_02599_b200.modules import SharedDecodeModule

    B, ctx = 6, [17, 40, 5, 33, 64, 21]
    kv = KvPool(spec, sum(pages_for(c + steps + 1) for c in ctx) + 2, cuda)
    kv.fill_random_(7)
    dec = SharedDecodeModule(spec, dw, kv, B, 128)
    bt = torch.zeros(B, dec.max_pages, dtype=torch.int32)
    nxt = 0
    for i, c in enumerate(ctx):
        n = pages_for(c + steps + 1)
        bt[i, :n] = torch.arange(nxt, nxt + n, dtype=torch.int32)
        nxt += n
    toks = torch.tensor([3, 99, 7, 250, 1, 42], dtype=torch.int32)
    out = []
    for t in range(steps):
        toks = dec.decode(toks, torch.tensor(ctx, dtype=torch.int32) + t, bt).cpu()
        out.append(dec.logits[:B].cpu().clone())
    return torch.stack(out)


@pytest.mark.parametrize("bias", [False, True])
def test_w4_module_from_ct_and_sunckpt_bit_identical(cuda, tmp_path, bias):
    from paper_2603_02599_b200 import checkpoint
    from paper_2603_02599_b200.spec import TINY
    from paper_2603_02599_b200.weights import DeviceWeights, init_weights

    spec = replace(TINY, name="tiny", ffn=768, qkv_bias=bias)  # W4 needs K % 128 == 0
    w = init_weights(spec, seed=5)
    spec4 = spec.with_bits(4)
    ref = DeviceWeights(spec4, w, cuda, 128)
    imp = checkpoint.from_compressed_tensors(spec, _ct_state(spec, w), cuda, 128)
    path = tmp_path / "m.sunckpt"
    checkpoint.save(path, imp)
    back = checkpoint.load(path, cuda, 128)
    torch.cuda.synchronize()
    for other in (imp, back):
        for (n1, a), (n2, b) in zip(checkpoint._named_tensors(ref), checkpoint._named_tensors(other)):
            assert n1 == n2 and torch.equal(a.view(torch.uint8), b.view(torch.uint8)), n1
    l_ref = _decode_logits(spec4, ref, cuda)
    assert torch.isfinite(l_ref).all()
    assert torch.equal(l_ref, _decode_logits(spec4, imp, cuda))
    assert torch.equal(l_ref, _decode_logits(spec4, back, cuda))
