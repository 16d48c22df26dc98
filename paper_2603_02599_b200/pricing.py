"""Decode-step pricing: the reference's analytic operator and the B200 backend.

The reference prices a decode iteration as ``D + (W_dec + sum_i tokens_i *
kvb) / (mbu * BW)`` (/root/reference/pkg/src/poolsim/costmodel.py:101-140),
called once per step at engine.py:427-429. That call site is the plugin
boundary of the shared decode path; ``DecodeBackend`` names it:

* ``AnalyticBackend`` — the reference formula (same signatures, same
  ``MixedDecoderError`` / ``ValueError`` behaviour);
* ``MeasuredBackend`` — the B200's measured step time over a (batch, context)
  grid (scripts/measure_step_grid.py, tests/golden/b200_steps_*.json), so the
  simulator predicts the new system (harness closure);
* ``calibrate_decode`` — the decode half of the reference's ``calibrate``
  (costmodel.py:257-358) refit to B200-measured concurrency-1 TPOT.

``step_bytes`` is the algorithmic-bytes model used for every roofline number
this package reports.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass
from typing import Iterable, Protocol

import bisect
import csv
import json

import numpy as np

from .errors import CalibrationInfeasible, MixedDecoderError
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
    """What a decode worker calls once per step (engine.py:427-429). ``batch``
    (the post-admission batch size) is extra information a backend may use."""

    def step_time(self, total_kv_bytes: float, decoder_weight_bytes: float, batch: int | None = None) -> float: ...


class AnalyticBackend:
    """The reference's closed form, unchanged."""

    def __init__(self, params: CostParams, gpu: GpuSpec):
        self.params, self.gpu = params, gpu

    def step_time(self, total_kv_bytes: float, decoder_weight_bytes: float, batch: int | None = None) -> float:
        return decode_step_time_from_totals(total_kv_bytes, decoder_weight_bytes, self.params, self.gpu)


# --------------------------------------------------------------------------- calibration (costmodel.py:186-358)
FLOPS_PER_PARAM = 2.0


def single_request_ttft(model: ModelProfile, isl: int, params: CostParams, gpu: GpuSpec) -> float:
    """Closed-form TTFT of an unqueued single request: prefill + transfer (costmodel.py:186-191)."""
    kv = KvHandle(request_id=-1, resident_tokens=isl, bytes_per_token=model.kv_bytes_per_token)
    return prefill_time(model, isl, params, gpu) + transfer_time(kv, gpu)


@dataclass(frozen=True)
class CalibrationTarget:
    """One measured concurrency-1 operating point (costmodel.py:194-210)."""

    param_count: float
    kv_bytes_per_token: int
    prefill_bits: int
    decode_bits: int
    isl: int
    osl: int
    ttft_s: float | None = None
    tpot_s: float | None = None
    label: str = ""


def load_targets_csv(path: str, param_count: float, kv_bytes_per_token: int) -> list[CalibrationTarget]:
    """costmodel.py:213-243: columns model, prefill_bits, decode_bits, isl, osl,
    concurrency, ttft_ms, tpot_ms; rows at concurrency != 1 are skipped."""
    out = []
    with open(path, newline="") as fh:
        for row in csv.DictReader(fh):
            if int(row["concurrency"]) != 1:
                continue
            ttft, tpot = row.get("ttft_ms", "").strip(), row.get("tpot_ms", "").strip()
            out.append(CalibrationTarget(param_count=param_count, kv_bytes_per_token=kv_bytes_per_token,
                                         prefill_bits=int(row["prefill_bits"]), decode_bits=int(row["decode_bits"]),
                                         isl=int(row["isl"]), osl=int(row["osl"]),
                                         ttft_s=float(ttft) / 1000.0 if ttft else None,
                                         tpot_s=float(tpot) / 1000.0 if tpot else None, label=row.get("model", "")))
    return out


def _target_profile(t: CalibrationTarget) -> ModelProfile:
    return ModelProfile(model_id=0, param_count=t.param_count, prefill_weight_bits=t.prefill_bits,
                        decode_weight_bits=t.decode_bits, kv_bytes_per_token=t.kv_bytes_per_token)


def calibrate(targets: list[CalibrationTarget], gpu: GpuSpec, rel_tol: float = 0.03) -> CostParams:
    """The reference's fit (costmodel.py:257-358): closed-form least squares of
    TTFT - transfer = F + c*isl (c -> penalised q for low-bit prefill) and of
    TPOT = D + beta * (W + mean resident KV bytes); mfu / mbu from the slopes;
    ``CalibrationInfeasible`` on too few targets, unphysical constants or a
    target reproduced worse than rel_tol. ``calibrate_decode`` below refits the
    decode half to B200-measured whole steps instead."""
    if len(targets) < 2:
        raise CalibrationInfeasible("need at least 2 targets spanning both precisions")
    ttft_rows = [t for t in targets if t.ttft_s is not None]
    tpot_rows = [t for t in targets if t.tpot_s is not None]
    if not ttft_rows or not tpot_rows:
        raise CalibrationInfeasible("targets must include at least one TTFT and one TPOT")
    lowbit = any(t.prefill_bits < 16 for t in ttft_rows)
    a = np.zeros((len(ttft_rows), 3 if lowbit else 2))
    z = np.zeros(len(ttft_rows))
    for i, t in enumerate(ttft_rows):
        z[i] = t.ttft_s - transfer_time(KvHandle(request_id=-1, resident_tokens=t.isl,
                                                 bytes_per_token=t.kv_bytes_per_token), gpu)
        a[i, 0] = 1.0
        a[i, 2 if t.prefill_bits < 16 else 1] = t.isl
    sol, *_ = np.linalg.lstsq(a, z, rcond=None)
    overhead_p, per_token = float(sol[0]), float(sol[1])
    penalty = float(sol[2] / sol[1]) if lowbit and sol[1] != 0 else 1.0
    a2 = np.zeros((len(tpot_rows), 2))
    y2 = np.zeros(len(tpot_rows))
    for i, t in enumerate(tpot_rows):
        a2[i] = (1.0, t.param_count * t.decode_bits / 8.0 + mean_decode_resident_tokens(t.isl, t.osl)
                 * t.kv_bytes_per_token)
        y2[i] = t.tpot_s
    sol2, *_ = np.linalg.lstsq(a2, y2, rcond=None)
    overhead_d, beta = float(sol2[0]), float(sol2[1])
    if per_token <= 0 or beta <= 0:
        raise CalibrationInfeasible("targets imply non-positive per-token cost; check TTFT/TPOT orderings")
    flops_per_token = FLOPS_PER_PARAM * targets[0].param_count
    mfu = flops_per_token / (per_token * gpu.flops)
    if mfu > 1.0:
        mfu, flops_per_token = 1.0, per_token * gpu.flops
    mbu = 1.0 / (beta * gpu.hbm_bandwidth)
    if mbu > 1.0:
        raise CalibrationInfeasible(f"decode targets imply {1.0 / beta:.3e} B/s effective bandwidth, above "
                                    f"the GPU peak {gpu.hbm_bandwidth:.3e} B/s")
    params = CostParams(prefill_flops_per_token=flops_per_token, prefill_fixed_overhead=overhead_p,
                        decode_fixed_overhead=overhead_d, dequant_compute_penalty=max(penalty, 1.0), mfu=mfu, mbu=mbu)
    problems = params.validate()
    if problems:
        raise CalibrationInfeasible("fit produced invalid parameters: " + "; ".join(problems))
    res = []
    for t in targets:
        prof = _target_profile(t)
        name = t.label or f"{t.prefill_bits}/{t.decode_bits}@isl{t.isl}"
        if t.ttft_s is not None:
            res.append((f"{name}.ttft", (single_request_ttft(prof, t.isl, params, gpu) - t.ttft_s) / t.ttft_s))
        if t.tpot_s is not None:
            res.append((f"{name}.tpot", (single_request_tpot(prof, t.isl, t.osl, params, gpu) - t.tpot_s) / t.tpot_s))
    worst = max(abs(e) for _, e in res)
    if worst > rel_tol:
        raise CalibrationInfeasible(f"best fit misses tolerance {rel_tol:.1%} (worst {worst:.2%})",
                                    residuals=sorted(res, key=lambda r: -abs(r[1])))
    return params


# --------------------------------------------------------------------------- harness closure
@dataclass(frozen=True)
class StepPoint:
    """One measured B200 decode step: `batch` members, each with `context`
    resident tokens before the step, took `step_s` seconds."""

    batch: int
    context: int
    step_s: float


def load_step_points(path: str) -> tuple[dict, list[StepPoint]]:
    """tests/golden/b200_steps_*.json (scripts/measure_step_grid.py) -> (header, points)."""
    with open(path) as f:
        data = json.load(f)
    pts = [StepPoint(int(p["batch"]), int(p["context"]), float(p["step_s"])) for p in data["points"]]
    return {k: v for k, v in data.items() if k != "points"}, pts


def calibrate_decode(points: list[StepPoint], decoder_weight_bytes: float, kv_bytes_per_token: float, gpu: GpuSpec,
                     rel_tol: float = 0.03) -> tuple[float, float, list[tuple[str, float]]]:
    """Decode half of the reference's ``calibrate`` (costmodel.py:306-317, 335-358):
    least squares of tpot = D + beta * (W + resident KV bytes) over the targets,
    mbu = 1 / (beta * BW). Returns (decode_fixed_overhead, mbu, residuals);
    raises ``CalibrationInfeasible`` like the reference (too few targets, beta <= 0,
    mbu > 1, or a target missed by more than rel_tol). The reference fits
    concurrency-1 targets; points here are whole decode steps at any batch."""
    if len(points) < 2:
        raise CalibrationInfeasible("need at least 2 decode targets")
    a = np.zeros((len(points), 2))
    y = np.zeros(len(points))
    for i, p in enumerate(points):
        a[i] = (1.0, decoder_weight_bytes + p.batch * p.context * kv_bytes_per_token)
        y[i] = p.step_s
    (d, beta), *_ = np.linalg.lstsq(a, y, rcond=None)
    if beta <= 0:
        raise CalibrationInfeasible("targets imply non-positive seconds per byte")
    mbu = 1.0 / (beta * gpu.hbm_bandwidth)
    if mbu > 1.0:
        raise CalibrationInfeasible(f"decode targets imply {1.0 / beta:.3e} B/s effective bandwidth, above "
                                    f"the GPU peak {gpu.hbm_bandwidth:.3e} B/s")
    res = []
    for p in points:
        pred = d + beta * (decoder_weight_bytes + p.batch * p.context * kv_bytes_per_token)
        res.append((f"B{p.batch}@ctx{p.context}.tpot", (pred - p.step_s) / p.step_s))
    worst = max(abs(e) for _, e in res)
    if worst > rel_tol:
        raise CalibrationInfeasible(f"best fit misses tolerance {rel_tol:.1%} (worst {worst:.2%})",
                                    residuals=sorted(res, key=lambda r: -abs(r[1])))
    return float(d), float(mbu), res


class MeasuredBackend:
    """Decode-step price from the B200's own measurements: bilinear in (batch,
    mean resident context) over a measured grid, linear extrapolation in context
    beyond it (KV bytes are linear in context), clamped to the batch range.
    Drop-in for ``AnalyticBackend`` at engine.py:427 when the post-admission
    batch size is passed."""

    def __init__(self, points: list[StepPoint], kv_bytes_per_token: float):
        if not points:
            raise ValueError("MeasuredBackend needs at least one measured point")
        self.kvb = float(kv_bytes_per_token)
        self.batches = sorted({p.batch for p in points})
        self.contexts = sorted({p.context for p in points})
        grid = {(p.batch, p.context): p.step_s for p in points}
        missing = [(b, c) for b in self.batches for c in self.contexts if (b, c) not in grid]
        if missing:
            raise ValueError(f"measured grid incomplete, missing {missing[:4]}")
        self.t = np.array([[grid[(b, c)] for c in self.contexts] for b in self.batches])

    @staticmethod
    def _bracket(xs: list[int], x: float) -> tuple[int, int, float]:
        if len(xs) == 1:
            return 0, 0, 0.0
        i = min(max(bisect.bisect_right(xs, x) - 1, 0), len(xs) - 2)
        return i, i + 1, (x - xs[i]) / (xs[i + 1] - xs[i])

    def predict(self, batch: int, context: float) -> float:
        b = min(max(float(batch), self.batches[0]), self.batches[-1])
        i0, i1, fb = self._bracket(self.batches, b)
        j0, j1, fc = self._bracket(self.contexts, float(context))  # fc may fall outside [0, 1]: extrapolate
        row = lambda i: self.t[i, j0] + fc * (self.t[i, j1] - self.t[i, j0])  # noqa: E731
        return float(max(row(i0) + fb * (row(i1) - row(i0)), 0.0))

    def step_time(self, total_kv_bytes: float, decoder_weight_bytes: float, batch: int | None = None) -> float:
        if not batch:
            raise ValueError("MeasuredBackend needs the batch size")
        return self.predict(batch, total_kv_bytes / (batch * self.kvb))
