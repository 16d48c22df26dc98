"""Value types of the shared decode path, API-compatible with poolsim's domain
layer (/root/reference/pkg/src/poolsim/domain.py).

Same names, fields, defaults, enum values and error behaviour as the
reference, so code written against ``poolsim`` keeps working; the B200 path
adds physical state where the reference only counts tokens:

* ``KvHandle`` (domain.py:96-113) gains ``pages`` — the block-table row of the
  request's cache in the shared paged pool — and ``model_id`` (the task prefill
  module that produced it; the decode side never reads it).
* ``GpuSpec.b200()`` returns the pool's measured B200 figures (the reference's
  defaults, domain.py:136-144, describe an A100 and stay the default).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .errors import InvalidConfig

IN_TRANSIT = -1  # KvHandle.location while the cache is on the wire / awaiting admission (domain.py:14)


class PoolMode(str, Enum):
    ISOLATED = "isolated"
    SHARED = "shared"


class WorkerRole(str, Enum):
    PREFILL = "prefill"
    DECODE = "decode"


class RequestOutcome(str, Enum):
    IN_FLIGHT = "in_flight"
    COMPLETED = "completed"
    OVER_CAPACITY = "over_capacity"


class DecodeRule(str, Enum):
    PINNED = "pinned"
    LEAST_OUTSTANDING_TOKENS = "least_outstanding_tokens"
    ROUND_ROBIN = "round_robin"
    WEIGHTED_RANDOM = "weighted_random"


@dataclass
class Request:
    """One inference job: arrival -> prefill -> KV hand-off -> shared decode (domain.py:45-93)."""

    id: int
    model_id: int
    arrival_time: float
    isl: int
    target_osl: int
    realized_osl: int = 0
    prefill_start: float | None = None
    prefill_end: float | None = None
    transfer_end: float | None = None
    first_token_time: float | None = None
    completion_time: float | None = None
    outcome: RequestOutcome = RequestOutcome.IN_FLIGHT

    def __post_init__(self):
        for name in ("isl", "target_osl"):
            if getattr(self, name) < 1:
                raise ValueError(f"request {self.id}: {name} must be >= 1, got {getattr(self, name)}")

    @property
    def completed(self) -> bool:
        return self.outcome is RequestOutcome.COMPLETED

    def timestamp_chain(self) -> list[float]:
        chain = [self.arrival_time, self.prefill_start, self.prefill_end, self.transfer_end,
                 self.first_token_time, self.completion_time]
        if None in chain:
            raise ValueError(f"request {self.id} has an incomplete timestamp chain")
        return chain  # type: ignore[return-value]


@dataclass
class KvHandle:
    """A request's KV cache: token count + (on the B200 path) its physical pages."""

    request_id: int
    resident_tokens: int
    bytes_per_token: int
    location: int = IN_TRANSIT
    pages: list[int] = field(default_factory=list)
    model_id: int = -1

    @property
    def resident_bytes(self) -> int:
        return self.resident_tokens * self.bytes_per_token


@dataclass(frozen=True)
class ModelProfile:
    """One deployed (task) model; decode_weight_bits=4 is QSUN (domain.py:116-133)."""

    model_id: int
    param_count: float
    prefill_weight_bits: int = 16
    decode_weight_bits: int = 16
    kv_bytes_per_token: int = 131072
    shared_decoder: bool = False

    def weight_bytes(self, phase: WorkerRole) -> float:
        bits = self.decode_weight_bits if phase is WorkerRole.DECODE else self.prefill_weight_bits
        return self.param_count * bits / 8.0


_GPU_FIELDS = ("flops", "hbm_bandwidth", "hbm_capacity", "interconnect_bandwidth", "interconnect_latency")


@dataclass(frozen=True)
class GpuSpec:
    flops: float = 3.12e14
    hbm_bandwidth: float = 2.039e12
    hbm_capacity: float = 8.0e10
    interconnect_bandwidth: float = 6.4e10
    interconnect_latency: float = 2.0e-4

    def validate(self, path: str = "gpu") -> list[str]:
        return [f"{path}.{n}: must be > 0, got {getattr(self, n)}" for n in _GPU_FIELDS if not getattr(self, n) > 0]

    @classmethod
    def b200(cls, hbm_gbs: float | None = None, bf16_tflops: float | None = None,
             peaks_path: str | None = None) -> "GpuSpec":
        """B200 with the driver-measured HBM copy bandwidth and bf16 GEMM burst
        (MEASURED_PEAKS.json at the repo root; B200_PROFILING.md's fallback 6.65 TB/s
        and 1.59 PFLOP/s when absent), NVLink-5 peer copy 770 GB/s, 180 GB."""
        import json
        import os

        if hbm_gbs is None or bf16_tflops is None:
            path = peaks_path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "MEASURED_PEAKS.json")
            try:
                with open(path) as f:
                    peaks = json.load(f)
                m_hbm, m_tf = float(peaks["hbm_gbs"]), float(peaks["bf16_tflops"])
            except (OSError, KeyError, ValueError):
                m_hbm, m_tf = 6650.0, 1590.0
            hbm_gbs = m_hbm if hbm_gbs is None else hbm_gbs
            bf16_tflops = m_tf if bf16_tflops is None else bf16_tflops
        return cls(flops=bf16_tflops * 1e12, hbm_bandwidth=hbm_gbs * 1e9, hbm_capacity=1.8e11,
                   interconnect_bandwidth=7.7e11, interconnect_latency=1.0e-5)


@dataclass
class WorkerState:
    worker_id: int
    role: WorkerRole
    served_models: frozenset[int]
    gpu: GpuSpec
    resident_kv_tokens: int = 0
    queue: list[int] = field(default_factory=list)
    active_batch: set[int] = field(default_factory=set)
    busy_until: float = 0.0


@dataclass(frozen=True)
class RoutingPolicy:
    decode_rule: DecodeRule = DecodeRule.LEAST_OUTSTANDING_TOKENS
    seed: int = 0
    load_metric: str = "anticipatory"  # or "kv_only"


@dataclass(frozen=True)
class ClusterConfig:
    models: tuple[ModelProfile, ...]
    decode_pool_mode: PoolMode
    decode_pool_size: int
    routing_policy: RoutingPolicy = RoutingPolicy()
    gpu_spec: GpuSpec = GpuSpec()

    @property
    def n_models(self) -> int:
        return len(self.models)

    @property
    def n_gpus_total(self) -> int:
        return self.n_models + self.decode_pool_size

    def decode_weight_bytes(self, model: ModelProfile) -> float:
        return model.weight_bytes(WorkerRole.DECODE)


def _model_checks(i: int, m: ModelProfile, seen: set) -> list[str]:
    p = f"cluster.models[{i}]"
    out = []
    if m.model_id in seen:
        out.append(f"{p}.model_id: duplicate id {m.model_id}")
    seen.add(m.model_id)
    if not m.param_count > 0:
        out.append(f"{p}.param_count: must be > 0, got {m.param_count}")
    for phase in ("prefill", "decode"):
        bits = getattr(m, f"{phase}_weight_bits")
        if bits not in (16, 4):
            out.append(f"{p}.{phase}_weight_bits: must be 16 or 4, got {bits}")
    if not m.kv_bytes_per_token > 0:
        out.append(f"{p}.kv_bytes_per_token: must be > 0, got {m.kv_bytes_per_token}")
    return out


def validate_cluster(config: ClusterConfig) -> ClusterConfig:
    """All structural invariants at once (domain.py:228-318); raises InvalidConfig.

    The shared-decoder invariant (every shared model agrees on decode bits and
    param count — one parameter set) is what makes a mixed-model batch legal.
    """
    problems: list[str] = []
    if not config.models:
        problems.append("cluster.models: at least one model is required")
    if config.decode_pool_size < 1:
        problems.append(f"cluster.decode_pool_size: must be >= 1, got {config.decode_pool_size}")
    problems += config.gpu_spec.validate("cluster.gpu")
    seen: set = set()
    for i, m in enumerate(config.models):
        problems += _model_checks(i, m, seen)

    shared = [m for m in config.models if m.shared_decoder]
    if shared:
        for attr, label in (("decode_weight_bits", "decode_weight_bits"), ("param_count", "param_count")):
            vals = sorted({getattr(m, attr) for m in shared})
            if len(vals) > 1:
                tail = "; a shared decoder has one parameter set" if attr == "decode_weight_bits" else ""
                problems.append(f"cluster.models: shared_decoder models disagree on {label} {vals}{tail}")

    rule = config.routing_policy.decode_rule
    if config.decode_pool_mode is PoolMode.ISOLATED:
        if config.decode_pool_size != len(config.models):
            problems.append("cluster.decode_pool_size: isolated mode requires one decode worker per model "
                            f"(K == {len(config.models)}), got {config.decode_pool_size}")
        if rule is not DecodeRule.PINNED:
            problems.append(f"cluster.routing_policy.decode_rule: isolated mode requires 'pinned', got '{rule.value}'")
    else:
        loose = [m.model_id for m in config.models if not m.shared_decoder]
        if loose:
            problems.append("cluster.models: shared pool mode requires shared_decoder=true for all models; "
                            f"models {loose} are not marked shared")
        if rule is DecodeRule.PINNED:
            problems.append("cluster.routing_policy.decode_rule: 'pinned' is only legal in isolated mode")

    cap = config.gpu_spec.hbm_capacity
    for i, m in enumerate(config.models):
        for phase in (WorkerRole.PREFILL, WorkerRole.DECODE):
            if m.weight_bytes(phase) > cap:
                problems.append(f"cluster.models[{i}]: {phase.value} weights exceed gpu.hbm_capacity")
    if problems:
        raise InvalidConfig(problems)
    return config


# Worker-id layout (domain.py:321-334): prefill workers 0..N-1 by model id,
# decode workers N..N+K-1; isolated mode pins model i to decode worker N+i.
def prefill_worker_id(model_id: int) -> int:
    return model_id


def decode_worker_ids(config: ClusterConfig) -> list[int]:
    return [config.n_models + k for k in range(config.decode_pool_size)]


def pinned_decode_worker(config: ClusterConfig, model_id: int) -> int:
    return config.n_models + model_id
