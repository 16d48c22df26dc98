"""Virtual-clock replay: the B200 serving loop (scheduler.py) with the
reference's analytic step price reproduces the reference simulator's dispatch
sequence, per-step batch sizes and charged KV bytes exactly
(engine_golden.json, made from poolsim.engine.run by tests/golden/make_golden.py),
plus the reference engine's closed-form known answers (pkg/tests/test_engine.py)."""
import json
import os

import pytest

from paper_2603_02599_b200 import pricing, scheduler
from paper_2603_02599_b200.sun_types import (ClusterConfig, DecodeRule, GpuSpec, KvHandle, ModelProfile, PoolMode,
                                             Request, RequestOutcome, RoutingPolicy, WorkerRole)
from paper_2603_02599_b200.trace import WorkloadSpec, generate_trace

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
COST = pricing.CostParams(prefill_flops_per_token=2.0e10, prefill_fixed_overhead=0.01, decode_fixed_overhead=0.002,
                          dequant_compute_penalty=1.25, mfu=0.5, mbu=0.8)
GPU = GpuSpec(flops=1.0e14, hbm_bandwidth=1.0e12, hbm_capacity=8.0e10, interconnect_bandwidth=5.0e10,
              interconnect_latency=1.0e-4)


def cluster(n_models, pool, rule, gpu=GPU):
    mode = PoolMode.ISOLATED if rule is DecodeRule.PINNED else PoolMode.SHARED
    models = tuple(ModelProfile(model_id=i, param_count=8.03e9, kv_bytes_per_token=131072,
                                shared_decoder=mode is PoolMode.SHARED) for i in range(n_models))
    return ClusterConfig(models=models, decode_pool_mode=mode, decode_pool_size=pool,
                         routing_policy=RoutingPolicy(decode_rule=rule, seed=3), gpu_spec=gpu)


def test_replay_matches_reference_engine_exactly():
    runs = json.load(open(os.path.join(GOLDEN, "engine_golden.json")))["runs"]
    for run in runs:
        sp = run["spec"]
        rule = DecodeRule(sp["rule"])
        cfg = cluster(sp["n_models"], sp["pool"], rule)
        ws = WorkloadSpec(n_models=sp["n_models"], total_rps=sp["rps"], alpha=sp["alpha"], isl=sp["isl"],
                          osl=sp["osl"], grace_period=1.0, measurement_window=4.0, seed=42)
        trace = generate_trace(ws)
        assert len(trace) == run["n_requests"]
        res = scheduler.run(cfg, trace, COST)
        assert [list(d) for d in res.log.dispatches] == run["dispatches"], sp
        assert [[w, b, kvb] for (w, _t, _d, b, kvb) in res.log.steps] == run["steps"], sp
        assert res.log.charged_steps == run["charged_steps"]


def test_event_trace_and_summary_match_reference_engine():
    """record_events=True gives the reference's event trace (engine.py:71-81, 301-303)
    entry for entry, and summarize(window, cluster, spec) (metrics.py:102-150) the
    reference's RunSummary field for field, on the same runs."""
    from paper_2603_02599_b200.stats import summarize
    from paper_2603_02599_b200.trace import measurement_filter

    runs = json.load(open(os.path.join(GOLDEN, "engine_golden.json")))["runs"]
    for run in runs:
        sp = run["spec"]
        cfg = cluster(sp["n_models"], sp["pool"], DecodeRule(sp["rule"]))
        ws = WorkloadSpec(n_models=sp["n_models"], total_rps=sp["rps"], alpha=sp["alpha"], isl=sp["isl"],
                          osl=sp["osl"], grace_period=1.0, measurement_window=4.0, seed=42)
        res = scheduler.run(cfg, generate_trace(ws), COST, None, None, True)
        assert res.resource_log is res.log
        got = [[round(t * 1e9), k.name, rid, wid] for (t, k, rid, wid) in res.event_trace]
        assert got == run["events"], sp
        summ = summarize(measurement_filter(res.completed, ws), cfg, ws).to_dict()
        assert summ == run["summary"], sp


def test_single_request_chain_closed_form():
    cfg = cluster(1, 1, DecodeRule.LEAST_OUTSTANDING_TOKENS)
    m = cfg.models[0]
    res = scheduler.run(cfg, [Request(id=0, model_id=0, arrival_time=0.5, isl=1024, target_osl=8)], COST)
    done = res.completed[0]
    t = 0.5 + pricing.prefill_time(m, 1024, COST, GPU)
    assert done.prefill_end == pytest.approx(t, abs=1e-9)
    t += pricing.transfer_time(KvHandle(0, 1024, m.kv_bytes_per_token), GPU)
    assert done.first_token_time == done.transfer_end == pytest.approx(t, abs=1e-9)
    w = m.weight_bytes(WorkerRole.DECODE)
    for k in range(7):
        t += pricing.decode_step_time([(m, 1024 + k)], w, COST, GPU)
    assert done.completion_time == pytest.approx(t, abs=1e-9)
    assert res.log.charged_steps == 7 and done.realized_osl == 8


def test_capacity_gated_admission_and_reject():
    # capacity fits the weights + two members' final KV only
    models = tuple(ModelProfile(i, 8.03e9, shared_decoder=True) for i in range(4))
    w = models[0].weight_bytes(WorkerRole.DECODE)
    res_bytes = (1024 + 8 - 1) * 131072
    gpu = GpuSpec(flops=1.0e14, hbm_bandwidth=1.0e12, hbm_capacity=w + 2 * res_bytes + 1,
                  interconnect_bandwidth=5.0e10, interconnect_latency=1.0e-4)
    cfg = ClusterConfig(models=models, decode_pool_mode=PoolMode.SHARED, decode_pool_size=1, gpu_spec=gpu)
    # four task models prefill in parallel, their KV lands together on the one shared decode GPU
    trace = [Request(id=i, model_id=i, arrival_time=0.0, isl=1024, target_osl=8) for i in range(4)]
    trace.append(Request(id=4, model_id=0, arrival_time=0.0, isl=400000, target_osl=8))  # can never fit
    res = scheduler.run(cfg, trace, COST)
    assert max(b for (_w, _t, _d, b, _k) in res.log.steps) == 2
    assert res.log.rejected_ids == [4]
    assert res.requests[4].outcome is RequestOutcome.OVER_CAPACITY
    assert sorted(res.log.freed_request_ids) == [0, 1, 2, 3, 4]
    assert res.log.charged_steps == 4 * 7


def test_token_conservation_random_configs():
    import random

    rng = random.Random(7)
    for _ in range(25):
        n = rng.randint(1, 6)
        rule = rng.choice([DecodeRule.LEAST_OUTSTANDING_TOKENS, DecodeRule.ROUND_ROBIN, DecodeRule.WEIGHTED_RANDOM])
        cfg = cluster(n, rng.randint(1, 4), rule)
        ws = WorkloadSpec(n_models=n, total_rps=rng.uniform(1, 20), alpha=rng.choice([0.0, 1.5, 3.0]),
                          isl=rng.randint(1, 2048), osl=rng.randint(1, 128), grace_period=0.5,
                          measurement_window=2.0, seed=rng.randint(0, 99))
        trace = generate_trace(ws)
        res = scheduler.run(cfg, trace, COST)
        done = res.completed
        assert res.log.charged_steps == sum(r.realized_osl - 1 for r in done)
        assert res.log.kv_created == res.log.kv_freed == len(trace)
        for r in done:
            chain = r.timestamp_chain()
            assert chain == sorted(chain)


class _PagedExecutor:
    """CPU stand-in for B200Executor's physical admission: a page pool and a batch limit."""

    def __init__(self, pages, max_batch, max_context=10_000):
        from paper_2603_02599_b200.kvpool import PageAllocator

        self.alloc = PageAllocator(pages)
        self.max_batch, self.max_context = max_batch, max_context
        self.max_seen = 0

    def fits(self, m, batch):
        from paper_2603_02599_b200.kvpool import pages_for

        r = m.request
        need = pages_for(r.isl + r.target_osl - 1)
        if need > self.alloc.num_pages or r.isl + r.target_osl - 1 > self.max_context:
            return "never"
        if batch >= self.max_batch or need > self.alloc.free_pages:
            return "never" if batch == 0 else "wait"
        return "ok"

    def admit(self, m):
        from paper_2603_02599_b200.kvpool import pages_for

        m.kv.pages = self.alloc.alloc(pages_for(m.request.isl + m.request.target_osl - 1))

    def step(self, members):
        self.max_seen = max(self.max_seen, len(members))
        return [0] * len(members)

    def retire(self, m):
        self.alloc.free(m.kv.pages)


def test_physical_admission_blocks_and_rejects():
    """The executor's page pool / batch limit gate admission like the virtual HBM
    capacity does (head-of-line blocking, reject-if-never-fits): the loop never asks
    the GPU for more pages or rows than it has, and everything else completes."""
    cfg = cluster(1, 1, DecodeRule.LEAST_OUTSTANDING_TOKENS)
    trace = [Request(id=i, model_id=0, arrival_time=0.01 * i, isl=64, target_osl=17) for i in range(12)]
    trace.append(Request(id=12, model_id=0, arrival_time=0.2, isl=4000, target_osl=8))  # > the whole pool
    ex = _PagedExecutor(pages=20, max_batch=3)  # 5 pages per request: at most 3 resident (batch limit)
    res = scheduler.run(cfg, trace, COST, executors={1: ex})
    assert ex.max_seen <= 3
    assert res.log.rejected_ids == [12]
    assert len(res.completed) == 12 and ex.alloc.free_pages == 20
