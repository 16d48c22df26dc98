"""Decoder geometries of the BASELINE.json configs (random-init, synthetic).

BASELINE.json config 1 names a "reference tiny decoder (pkg/configs default)"
that does not exist in the reference: TINY is the substitute
from SURVEY.md §8(d) with head_dim 64 (the attention kernel implements
head_dim 64 and 128, the two sizes every named config uses) — a deliberate,
documented deviation from the survey's 8q/2kv x 32 sketch.
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class DecoderSpec:
    name: str
    vocab: int
    hidden: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float
    rms_eps: float = 1e-5
    qkv_bias: bool = False
    tie_embeddings: bool = False
    weight_bits: int = 16          # 16 = bf16 decode module; 4 = QSUN W4A16
    group_size: int = 128
    init_std: float = 0.02
    lm_head_std: float = 0.02
    # margin-engineered greedy (parity tests, SURVEY §7 hard part (b)): embedding rows
    # ~ N(0, embed_std) and lm_head row v = N(0, lm_head_std) + greedy_margin / (hidden *
    # embed_std) * embed[perm[v]] for a seeded permutation perm, so the logit of token
    # perm^-1(x) carries ~greedy_margin * rho (rho = embed_std / rms(final residual)) on
    # top of the random part: greedy decisions are far from ties while every logit still
    # depends on the whole layer stack. 0 = plain random init.
    embed_std: float | None = None
    greedy_margin: float = 0.0

    @property
    def kv_bytes_per_token(self) -> int:
        """2 (K,V) * L * n_kv * d * 2 bytes — ModelProfile.kv_bytes_per_token (domain.py:124)."""
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    @property
    def qkv_rows(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def gate_up_rows(self) -> int:
        return (self.ffn + 63) // 64 * 128

    def linear_shapes(self) -> dict[str, tuple[int, int]]:
        qd = self.n_q_heads * self.head_dim
        return {"qkv": (self.qkv_rows, self.hidden), "o": (self.hidden, qd),
                "gate_up": (self.gate_up_rows, self.hidden), "down": (self.hidden, self.ffn)}

    @property
    def param_count(self) -> int:
        """Parameters of the decode module (embedding + layers + final norm + lm_head)."""
        h, qd, kd = self.hidden, self.n_q_heads * self.head_dim, self.n_kv_heads * self.head_dim
        per_layer = h * (qd + 2 * kd) + qd * h + 3 * h * self.ffn + 2 * h
        if self.qkv_bias:
            per_layer += qd + 2 * kd
        lm = 0 if self.tie_embeddings else self.vocab * h
        return self.vocab * h + self.n_layers * per_layer + h + lm

    def decode_weight_bytes(self) -> int:
        """Bytes one decode step must stream: every linear layer + lm_head (+ W4
        group scales), excluding the embedding table (only B rows are read).
        SURVEY.md §8(d) `W_dec`."""
        h, qd, kd = self.hidden, self.n_q_heads * self.head_dim, self.n_kv_heads * self.head_dim
        lin = h * (qd + 2 * kd) + qd * h + 3 * h * self.ffn
        if self.weight_bits == 4:
            lin_bytes = lin // 2 + (lin // self.group_size) * 2
        else:
            lin_bytes = lin * 2
        norms = (2 * self.n_layers + 1) * h * 2
        bias = (qd + 2 * kd) * 2 * self.n_layers if self.qkv_bias else 0
        return self.n_layers * lin_bytes + norms + bias + self.vocab * h * 2

    def with_bits(self, bits: int) -> "DecoderSpec":
        return replace(self, weight_bits=bits, name=self.name + ("-w4" if bits == 4 else ""))


TINY = DecoderSpec("tiny", vocab=512, hidden=256, n_layers=4, n_q_heads=8, n_kv_heads=2, head_dim=64,
                   ffn=688, rope_theta=1e4, lm_head_std=0.05)
LLAMA32_1B = DecoderSpec("llama3.2-1b", vocab=128256, hidden=2048, n_layers=16, n_q_heads=32, n_kv_heads=8,
                         head_dim=64, ffn=8192, rope_theta=5e5, tie_embeddings=True)
LLAMA31_8B = DecoderSpec("llama3.1-8b", vocab=128256, hidden=4096, n_layers=32, n_q_heads=32, n_kv_heads=8,
                         head_dim=128, ffn=14336, rope_theta=5e5)
QWEN25_14B = DecoderSpec("qwen2.5-14b", vocab=152064, hidden=5120, n_layers=48, n_q_heads=40, n_kv_heads=8,
                         head_dim=128, ffn=13824, rope_theta=1e6, rms_eps=1e-6, qkv_bias=True)

SPECS = {s.name: s for s in (TINY, LLAMA32_1B, LLAMA31_8B, QWEN25_14B)}
