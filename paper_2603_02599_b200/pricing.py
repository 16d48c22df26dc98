"""Decode-step pricing: the reference's analytic operator and the B200 backend.

The reference prices a decode iteration as ``D + (W_dec + sum_i tokens_i *
kvb) / (mbu * BW)`` (/root/reference/pkg/src/poolsim/costmodel.py:101-140),
called once per step at engine.py:427-429. That call site is the plugin
boundary of the shared decode path; ``DecodeBackend`` names it:

* ``AnalyticBackend`` — the reference formula (same signatures, same
  ``MixedDecoderError`` / ``ValueError`` behaviour);
* ``paper_2603_02599_b200.scheduler.B200Backend`` — runs the real step on a B200
  and returns its measured duration.

``step_bytes`` is the algorithmic-bytes model used for every roofline number
this package reports.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass
from typing import Iterable, Protocol

from .errors import MixedDecoderError
from .spec import DecoderSpec
from .sun_types import GpuSpec, KvHandle, ModelProfile, WorkerRole


@dataclass(frozen=True)
class CostParams:
    """Calibrated constants of the analytic model (costmodel.py:40-83)."""

    prefill_flops_per_token: float
    prefill_fixed_overhead: float
    decode_fixed_overhead: float
    dequant_compute_penalty: float = 1.0
    mfu: float = 1.0
    mbu: float = 1.0

    def validate(self, path: str = "cost") -> list[str]:
        out = [f"{path}.{n}: must be > 0, got {getattr(self, n)}"
               for n in ("prefill_flops_per_token", "prefill_fixed_overhead", "decode_fixed_overhead", "mfu", "mbu")
               if not getattr(self, n) > 0]
        out += [f"{path}.{n}: must be <= 1, got {getattr(self, n)}" for n in ("mfu", "mbu") if not getattr(self, n) <= 1]
        if not self.dequant_compute_penalty >= 1.0:
            out.append(f"{path}.dequant_compute_penalty: must be >= 1, got {self.dequant_compute_penalty}")
        return out

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, data: dict) -> "CostParams":
        return cls(**data)


def prefill_time(model: ModelProfile, isl: int, params: CostParams, gpu: GpuSpec) -> float:
    """Analytic prefill price (costmodel.py:86-98): affine in prompt tokens, with
    the dequantisation penalty when prefill weights are low-bit. The prefill
    module is producer-side; the simulator uses this for its event times."""
    if isl < 1:
        raise ValueError(f"isl must be >= 1, got {isl}")
    penalty = params.dequant_compute_penalty if model.prefill_weight_bits < 16 else 1.0
    return params.prefill_fixed_overhead + penalty * (isl * params.prefill_flops_per_token / (params.mfu * gpu.flops))


def decode_step_time_from_totals(total_kv_bytes: float, decoder_weight_bytes: float, params: CostParams,
                                 gpu: GpuSpec) -> float:
    """Weights read once per step + the batch's KV, over effective bandwidth."""
    return params.decode_fixed_overhead + (decoder_weight_bytes + total_kv_bytes) / (params.mbu * gpu.hbm_bandwidth)


def _one_weight_set(members: list[tuple[ModelProfile, int]]) -> None:
    sets = {(m.param_count, m.decode_weight_bits) for m, _ in members}
    if len(sets) > 1:
        raise MixedDecoderError(f"batch members carry {len(sets)} distinct decoder weight sets")


def kv_step_bytes(batch: Iterable[tuple[ModelProfile, int]]) -> float:
    return sum(tokens * m.kv_bytes_per_token for m, tokens in batch)


def decode_step_time(batch: Iterable[tuple[ModelProfile, int]], decoder_weight_bytes: float, params: CostParams,
                     gpu: GpuSpec) -> float:
    members = list(batch)
    if not members:
        raise ValueError("decode batch must be non-empty")
    _one_weight_set(members)
    return decode_step_time_from_totals(kv_step_bytes(members), decoder_weight_bytes, params, gpu)


def transfer_time(kv: KvHandle, gpu: GpuSpec) -> float:
    """Prefill -> decode KV hand-off: latency + bytes / link bandwidth (costmodel.py:148-155)."""
    if kv.resident_tokens < 1:
        raise ValueError("cannot transfer an empty KV cache")
    return gpu.interconnect_latency + kv.resident_tokens * kv.bytes_per_token / gpu.interconnect_bandwidth


def mean_decode_resident_tokens(isl: int, osl: int) -> float:
    return float(isl) if osl < 2 else isl + (osl - 2) / 2.0


def single_request_tpot(model: ModelProfile, isl: int, osl: int, params: CostParams, gpu: GpuSpec,
                        decoder_weight_bytes: float | None = None) -> float:
    if osl < 2:
        raise ValueError("TPOT is undefined for osl < 2")
    w = model.weight_bytes(WorkerRole.DECODE) if decoder_weight_bytes is None else decoder_weight_bytes
    kv = mean_decode_resident_tokens(isl, osl) * model.kv_bytes_per_token
    return params.decode_fixed_overhead + (w + kv) / (params.mbu * gpu.hbm_bandwidth)


def step_bytes(spec: DecoderSpec, contexts: Iterable[int]) -> int:
    """Algorithmic HBM bytes of one B200 decode step:
    W_dec + sum_i ctx_i*kvb (KV read, ctx before append) + B*kvb (append)
    + B*h*2 (embedding rows) + B*V*4 (fp32 logits)."""
    ctx = list(contexts)
    b = len(ctx)
    kvb = spec.kv_bytes_per_token
    return spec.decode_weight_bytes() + sum(ctx) * kvb + b * kvb + b * spec.hidden * 2 + b * spec.vocab * 4


class DecodeBackend(Protocol):
    """What a decode worker calls once per step (engine.py:427-429)."""

    def step_time(self, total_kv_bytes: float, decoder_weight_bytes: float) -> float: ...


class AnalyticBackend:
    """The reference's closed form, unchanged."""

    def __init__(self, params: CostParams, gpu: GpuSpec):
        self.params, self.gpu = params, gpu

    def step_time(self, total_kv_bytes: float, decoder_weight_bytes: float) -> float:
        return decode_step_time_from_totals(total_kv_bytes, decoder_weight_bytes, self.params, self.gpu)
