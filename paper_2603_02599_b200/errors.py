"""Exception types, named after the reference's (poolsim) so callers' except
clauses keep working: ``MixedDecoderError`` (costmodel.py:27-28),
``EmptyPool``/``UnknownModel`` (routing.py:16-21), ``InvalidConfig``
(domain.py:33-42), ``CalibrationInfeasible`` (costmodel.py). The B200 path adds ``OverCapacity`` (a request or batch that
cannot fit the KV pool / workspace, the physical form of the reference's
OVER_CAPACITY outcome, engine.py:394-401) and ``SunCudaError``."""
from __future__ import annotations


class MixedDecoderError(Exception):
    """A decode batch mixed members that do not share one weight set."""


class InvalidConfig(Exception):
    """A cluster/workload configuration violates an invariant (all violations listed)."""

    def __init__(self, violations: list[str]):
        self.violations = violations
        super().__init__("; ".join(violations))


class UnknownModel(Exception):
    """A request named a model with no mapped prefill / pinned decode worker."""


class EmptyPool(Exception):
    """Decode routing was asked to pick from an empty pool."""


class CalibrationInfeasible(Exception):
    """A calibration fit misses its tolerance or implies unphysical constants
    (costmodel.py CalibrationInfeasible: message + per-target residuals)."""

    def __init__(self, message: str, residuals: list[tuple[str, float]] | None = None):
        self.residuals = residuals or []
        detail = "; ".join(f"{name}: {err:+.2%}" for name, err in self.residuals)
        super().__init__(message + (f" [{detail}]" if detail else ""))


class OverCapacity(Exception):
    """Not enough KV pages / workspace for the request or batch."""


class UnsupportedShape(Exception):
    """A decoder geometry outside what the sm_100a kernels implement."""


class SunCudaError(RuntimeError):
    """CUDA runtime/driver failure inside libsun_b200.so."""
