"""Pin the CPU oracle (oracle/decoder_ref.py, oracle/quant_ref.py).

The reference has no decoder numerics (parity unpinned), so the
oracle's *block definition* is pinned against an independent, widely used
implementation instead: with its bf16 storage roundings disabled it must
reproduce transformers' LlamaForCausalLM / Qwen2ForCausalLM logits on the same
weights. Its prefill/decode split must equal one full causal forward (Eq. 4:
C = C_X || C_y), and the SUN-W4 packing must round-trip exactly.
"""
import random
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import quant_ref
from oracle.decoder_ref import OracleDecoder, OracleSpec, argmax_lowest
from paper_2603_02599_b200.spec import TINY
from paper_2603_02599_b200.weights import init_weights


def ospec(spec):
    return OracleSpec(spec.vocab, spec.hidden, spec.n_layers, spec.n_q_heads, spec.n_kv_heads, spec.head_dim,
                      spec.ffn, spec.rope_theta, spec.rms_eps, spec.qkv_bias)


def hf_model(spec, w):
    transformers = pytest.importorskip("transformers")
    common = dict(vocab_size=spec.vocab, hidden_size=spec.hidden, intermediate_size=spec.ffn,
                  num_hidden_layers=spec.n_layers, num_attention_heads=spec.n_q_heads,
                  num_key_value_heads=spec.n_kv_heads, head_dim=spec.head_dim, rms_norm_eps=spec.rms_eps,
                  rope_theta=spec.rope_theta, tie_word_embeddings=False, max_position_embeddings=4096)
    if spec.qkv_bias:
        cfg = transformers.Qwen2Config(**common, use_sliding_window=False)
        model = transformers.Qwen2ForCausalLM(cfg)
    else:
        cfg = transformers.LlamaConfig(**common, attention_bias=False, mlp_bias=False)
        model = transformers.LlamaForCausalLM(cfg)
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"], "lm_head.weight": w["lm_head"]}
    for l in range(spec.n_layers):
        p = f"model.layers.{l}."
        sd[p + "input_layernorm.weight"] = w[f"l{l}.attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = w[f"l{l}.ffn_norm"]
        for a, b in (("q", "wq"), ("k", "wk"), ("v", "wv"), ("o", "wo")):
            sd[p + f"self_attn.{a}_proj.weight"] = w[f"l{l}.{b}"]
        if spec.qkv_bias:
            for a in "qkv":
                sd[p + f"self_attn.{a}_proj.bias"] = w[f"l{l}.b{a}"]
        sd[p + "mlp.gate_proj.weight"] = w[f"l{l}.wg"]
        sd[p + "mlp.up_proj.weight"] = w[f"l{l}.wu"]
        sd[p + "mlp.down_proj.weight"] = w[f"l{l}.wd"]
    model.load_state_dict({k: v.float() for k, v in sd.items()}, strict=False)
    return model.float().eval()


@pytest.mark.parametrize("bias", [False, True])
def test_oracle_block_matches_transformers(bias):
    spec = replace(TINY, qkv_bias=bias, n_layers=2)
    w = init_weights(spec, seed=3)
    model = hf_model(spec, w)
    r = random.Random(5)
    prompt = [r.randrange(spec.vocab) for _ in range(40)]
    with torch.no_grad():
        ref = model(torch.tensor([prompt])).logits[0, -1].float()
    o = OracleDecoder(ospec(spec), w, 64, round_bf16=False)
    got, _ = o.prefill(prompt)
    torch.testing.assert_close(got, ref, rtol=1e-4, atol=1e-4)


def test_prefill_plus_decode_equals_full_forward():
    """Eq. 4: decoding over the prefill module's cache == one causal pass (same θ)."""
    spec = TINY
    w = init_weights(spec, seed=0)
    o = OracleDecoder(ospec(spec), w, 128, round_bf16=False)
    r = random.Random(1)
    seq = [r.randrange(spec.vocab) for _ in range(30)]
    full, _ = o.forward(seq, 0, None)
    _, cache = o.prefill(seq[:20])
    lg = None
    for t in range(20, 30):
        lg, cache = o.decode(seq[t], t, cache)
    torch.testing.assert_close(lg, full, rtol=1e-5, atol=1e-5)


def test_argmax_lowest_index_on_ties():
    x = torch.tensor([[1.0, 3.0, 3.0, 2.0], [0.0, 0.0, 0.0, 0.0]])
    assert argmax_lowest(x).tolist() == [1, 0]


def test_sun_w4_pack_roundtrip_and_bounds():
    g = torch.Generator().manual_seed(0)
    w = (torch.randn(200, 512, generator=g) * 0.02).to(torch.bfloat16)
    w[3, 128:256] = 0
    q, s = quant_ref.quantize(w)
    assert int(q.min()) >= -8 and int(q.max()) <= 7
    assert float(s[3, 1]) == 0.0 and int(q[3, 128:256].abs().max()) == 0
    packed, scales = quant_ref.pack(q, s)
    assert packed.size == 256 * 512 // 2 and scales.shape == (2, 4, 128)
    assert torch.equal(quant_ref.unpack(packed, 200, 512), q)
    deq = quant_ref.dequantize(q, s).float()
    rel = ((deq - w.float()).norm() / w.float().norm()).item()
    assert rel < 0.12  # 4-bit symmetric g128 on Gaussian weights


def test_sun_w4_nibble_order():
    q = torch.arange(-8, 8, dtype=torch.int8).repeat(128, 8)[:128, :128].contiguous()
    s = torch.ones(128, 1, dtype=torch.bfloat16)
    packed, _ = quant_ref.pack(q, s)
    word = packed[:4].view(np.uint32)[0]
    elems = [int(x) for x in q[0, :8]]
    nib = [int((int(word) >> (4 * i)) & 0xF) for i in range(8)]
    assert [nib[quant_ref.NIBBLE_OF_ELEM[e]] - 8 for e in range(8)] == elems
