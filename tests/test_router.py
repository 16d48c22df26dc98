"""Model-agnostic decode routing is bit-exact with the reference (poolsim
routing.py:59-102): golden vectors generated from the reference by
tests/golden/make_golden.py, plus the reference's own known-answer tests
(pkg/tests/test_routing.py:37-103) restated."""
import json
import os

import pytest

from paper_2603_02599_b200.errors import EmptyPool, UnknownModel
from paper_2603_02599_b200.router import DecodeDispatcher, PoolSnapshot, outstanding_tokens, route_prefill
from paper_2603_02599_b200.sun_types import DecodeRule, Request, RoutingPolicy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def req(model_id=0, rid=0):
    return Request(id=rid, model_id=model_id, arrival_time=0.0, isl=128, target_osl=8)


def snap(w, resident=0, queued=0, remaining=0):
    return PoolSnapshot(w, resident, queued, remaining)


def _replay(policy, pinned, steps):
    d = DecodeDispatcher(policy, pinned_map=pinned)
    picks = []
    for st in steps:
        pool = [PoolSnapshot(*s) for s in st["pool"]]
        r = Request(id=st["request"][0], model_id=st["request"][1], arrival_time=0.0, isl=128, target_osl=8)
        picks.append(d.route(r, pool))
    return picks


def test_golden_router_sequences_bit_exact():
    cases = json.load(open(os.path.join(GOLDEN, "router_golden.json")))
    assert len(cases) == 4 * 2 * 3
    for c in cases:
        policy = RoutingPolicy(decode_rule=DecodeRule(c["rule"]), seed=c["seed"], load_metric=c["load_metric"])
        pinned = {int(k): v for k, v in c["pinned_map"].items()} or None
        assert _replay(policy, pinned, c["steps"]) == [s["pick"] for s in c["steps"]], c["rule"]


def test_router_view_of_reference_simulator_replays_bit_exact():
    """Snapshot sequences the reference engine itself presented to its router."""
    runs = json.load(open(os.path.join(GOLDEN, "engine_golden.json")))["runs"]
    for run in runs:
        rule = DecodeRule(run["spec"]["rule"])
        policy = RoutingPolicy(decode_rule=rule, seed=run["policy_seed"])
        pinned = None
        if rule is DecodeRule.PINNED:
            n = run["spec"]["n_models"]
            pinned = {m: n + m for m in range(n)}
        picks = _replay(policy, pinned, run["router_view"])
        assert picks == [s["pick"] for s in run["router_view"]]
        assert [[rid, w] for rid, w in run["dispatches"]] == [[s["request"][0], s["pick"]] for s in run["router_view"]]


class TestKnownAnswers:
    def test_lot_min_load_with_id_tiebreak(self):
        p = RoutingPolicy(decode_rule=DecodeRule.LEAST_OUTSTANDING_TOKENS)
        assert DecodeDispatcher(p).route(req(), [snap(0, 500), snap(1, 200), snap(2, 200)]) == 1
        assert DecodeDispatcher(p).route(req(), [snap(2, 10), snap(0, 10), snap(1, 10)]) == 0

    def test_anticipatory_vs_kv_only(self):
        pool = [snap(0, 100, 0, 500), snap(1, 300)]
        assert DecodeDispatcher(RoutingPolicy()).route(req(), pool) == 1
        assert DecodeDispatcher(RoutingPolicy(load_metric="kv_only")).route(req(), pool) == 0
        assert outstanding_tokens(pool[0]) == 600 and outstanding_tokens(pool[0], "kv_only") == 100

    def test_model_agnostic(self):
        d = DecodeDispatcher(RoutingPolicy())
        assert {d.route(req(model_id=m, rid=m), [snap(0, 9), snap(1, 5)]) for m in range(4)} == {1}

    def test_round_robin_cycles_in_id_order(self):
        d = DecodeDispatcher(RoutingPolicy(decode_rule=DecodeRule.ROUND_ROBIN))
        assert [d.route(req(rid=i), [snap(3), snap(5), snap(4)]) for i in range(6)] == [3, 4, 5, 3, 4, 5]

    def test_weighted_random_seeded(self):
        p = RoutingPolicy(decode_rule=DecodeRule.WEIGHTED_RANDOM, seed=9)
        pool = [snap(0, 0), snap(1, 10_000)]
        a = [DecodeDispatcher(p).route(req(rid=i), pool) for i in range(20)]
        d = DecodeDispatcher(p)
        b = [d.route(req(rid=i), pool) for i in range(20)]
        assert a == b  # (reference test_routing.py:76-88: first draws of fresh streams == one stream here)
        assert b.count(0) > b.count(1)

    def test_pinned_and_errors(self):
        d = DecodeDispatcher(RoutingPolicy(decode_rule=DecodeRule.PINNED), pinned_map={0: 4, 1: 5})
        assert d.route(req(model_id=0), [snap(4), snap(5)]) == 4
        assert d.route(req(model_id=1), [snap(4), snap(5)]) == 5
        with pytest.raises(UnknownModel):
            d.route(req(model_id=2), [snap(4)])
        with pytest.raises(EmptyPool):
            DecodeDispatcher(RoutingPolicy()).route(req(), [])
        assert route_prefill(req(model_id=2), {0: 0, 1: 1, 2: 2}) == 2
        with pytest.raises(UnknownModel):
            route_prefill(req(model_id=7), {0: 0})
