"""Model-specific prefill routing + model-agnostic decode routing.

API mirror of /root/reference/pkg/src/poolsim/routing.py (PoolSnapshot 24-36,
outstanding_tokens 39-46, route_prefill 49-56, DecodeDispatcher 59-102); each
rule is a small strategy object here. Decisions are bit-exact with the
reference on identical snapshot sequences (tests/test_router.py replays the
reference's golden vectors and dispatch logs): shared-pool rules never read
the request's model id, which is what lets one decode batch mix task models
(PAPER.md:231-241).
"""
from __future__ import annotations

import random
from dataclasses import dataclass

from .errors import EmptyPool, UnknownModel
from .sun_types import DecodeRule, Request, RoutingPolicy


@dataclass(frozen=True)
class PoolSnapshot:
    """Load of one decode worker at decision time (from real per-GPU counters)."""

    worker_id: int
    resident_kv_tokens: int
    queued_prompt_tokens: int
    remaining_target_tokens: int


def outstanding_tokens(snap: PoolSnapshot, load_metric: str = "anticipatory") -> int:
    if load_metric == "kv_only":
        return snap.resident_kv_tokens
    return snap.resident_kv_tokens + snap.queued_prompt_tokens + snap.remaining_target_tokens


def route_prefill(request: Request, prefill_map: dict[int, int]) -> int:
    """Fixed model -> prefill-worker map (each task has its own prefill module)."""
    worker = prefill_map.get(request.model_id)
    if worker is None:
        raise UnknownModel(f"request {request.id}: model {request.model_id} has no prefill worker")
    return worker


class _Pinned:
    def __init__(self, table: dict[int, int]):
        self.table = table

    def pick(self, request: Request, pool: list[PoolSnapshot]) -> int:
        if request.model_id not in self.table:
            raise UnknownModel(f"request {request.id}: model {request.model_id} has no pinned decode worker")
        return self.table[request.model_id]


class _LeastOutstanding:
    def __init__(self, metric: str):
        self.metric = metric

    def pick(self, request: Request, pool: list[PoolSnapshot]) -> int:
        best = pool[0]
        best_key = (outstanding_tokens(best, self.metric), best.worker_id)
        for snap in pool[1:]:
            key = (outstanding_tokens(snap, self.metric), snap.worker_id)
            if key < best_key:
                best, best_key = snap, key
        return best.worker_id


class _RoundRobin:
    def __init__(self):
        self.counter = 0

    def pick(self, request: Request, pool: list[PoolSnapshot]) -> int:
        ids = sorted(s.worker_id for s in pool)
        wid = ids[self.counter % len(ids)]
        self.counter += 1
        return wid


class _WeightedRandom:
    """Inverse-load weights 1/(1+load) over workers in id order, drawn with the
    run's seeded CPython Mersenne Twister (the stream is part of run state)."""

    def __init__(self, seed: int, metric: str):
        self.rng = random.Random(seed)
        self.metric = metric

    def pick(self, request: Request, pool: list[PoolSnapshot]) -> int:
        ordered = sorted(pool, key=lambda s: s.worker_id)
        w = [1.0 / (1.0 + outstanding_tokens(s, self.metric)) for s in ordered]
        return self.rng.choices(ordered, weights=w, k=1)[0].worker_id


class DecodeDispatcher:
    """Centralised decode dispatcher; owns the stateful rule (RR counter, RNG)."""

    def __init__(self, policy: RoutingPolicy, pinned_map: dict[int, int] | None = None):
        self.policy = policy
        self.pinned_map = pinned_map or {}
        rule = policy.decode_rule
        if rule is DecodeRule.PINNED:
            self._rule = _Pinned(self.pinned_map)
        elif rule is DecodeRule.LEAST_OUTSTANDING_TOKENS:
            self._rule = _LeastOutstanding(policy.load_metric)
        elif rule is DecodeRule.ROUND_ROBIN:
            self._rule = _RoundRobin()
        elif rule is DecodeRule.WEIGHTED_RANDOM:
            self._rule = _WeightedRandom(policy.seed, policy.load_metric)
        else:
            self._rule = None

    def route(self, request: Request, pool: list[PoolSnapshot]) -> int:
        if not pool:
            raise EmptyPool("decode pool is empty")
        if self._rule is None:
            raise ValueError(f"unknown decode rule: {self.policy.decode_rule}")
        return self._rule.pick(request, pool)
