"""Generate the golden fixtures that pin the host side of the shared decode
path to the reference implementation (poolsim, /root/reference/pkg/src).

Run HERE (the reference is importable in the build container, not on the GPU
box): ``python tests/golden/make_golden.py``. It imports poolsim read-only
(PYTHONDONTWRITEBYTECODE, no cwd writes into /root/reference) and records:

* router_golden.json   — DecodeDispatcher.route decisions for every rule /
  load metric / seed over seeded random PoolSnapshot sequences, plus the
  snapshot sequences the reference simulator itself presents to the router
  (captured by wrapping DecodeDispatcher.route during engine.run);
* workload_golden.json — zipf_split values and generate_trace text outputs;
* engine_golden.json   — ResourceLog.dispatches and per-step batch sizes /
  charged KV bytes of small simulated runs (the schedule a real decode
  backend must replay), plus decode_step_time /
  transfer_time / single_request_tpot values;
* cluster_golden.json  — validate_cluster violation lists.
"""
from __future__ import annotations

import io
import json
import os
import random
import sys

os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import poolsim  # noqa: E402
from poolsim import engine, metrics, routing  # noqa: E402
from poolsim.costmodel import (CostParams, decode_step_time, single_request_tpot,  # noqa: E402
                               transfer_time)
from poolsim.domain import (ClusterConfig, DecodeRule, GpuSpec, InvalidConfig, KvHandle,  # noqa: E402
                            ModelProfile, PoolMode, Request, RoutingPolicy, validate_cluster)
from poolsim.workload import (ArrivalProcess, WorkloadSpec, generate_trace, measurement_filter,  # noqa: E402
                              write_trace, zipf_split)

OUT = os.path.dirname(os.path.abspath(__file__))

SIMPLE_COST = CostParams(prefill_flops_per_token=2.0e10, prefill_fixed_overhead=0.01, decode_fixed_overhead=0.002,
                         dequant_compute_penalty=1.25, mfu=0.5, mbu=0.8)
SIMPLE_GPU = GpuSpec(flops=1.0e14, hbm_bandwidth=1.0e12, hbm_capacity=8.0e10, interconnect_bandwidth=5.0e10,
                     interconnect_latency=1.0e-4)


def snap_dict(s):
    return [s.worker_id, s.resident_kv_tokens, s.queued_prompt_tokens, s.remaining_target_tokens]


def router_cases():
    cases = []
    rng = random.Random(20260317)
    for rule in DecodeRule:
        for metric in ("anticipatory", "kv_only"):
            for seed in (0, 9, 12345):
                policy = RoutingPolicy(decode_rule=rule, seed=seed, load_metric=metric)
                ids = rng.sample(range(4, 20), rng.randint(1, 8))
                pinned = {m: rng.choice(ids) for m in range(6)} if rule is DecodeRule.PINNED else None
                d = routing.DecodeDispatcher(policy, pinned_map=pinned)
                steps = []
                for i in range(60):
                    pool = [routing.PoolSnapshot(w, rng.randint(0, 5000), rng.choice([0, rng.randint(0, 3000)]),
                                                 rng.randint(0, 4000)) for w in rng.sample(ids, len(ids))]
                    if rng.random() < 0.15:  # ties on load
                        pool = [routing.PoolSnapshot(s.worker_id, 100, 0, 0) for s in pool]
                    req = Request(id=i, model_id=rng.randrange(6), arrival_time=0.0, isl=128, target_osl=8)
                    steps.append({"request": [req.id, req.model_id], "pool": [snap_dict(s) for s in pool],
                                  "pick": d.route(req, pool)})
                cases.append({"rule": rule.value, "load_metric": metric, "seed": seed,
                              "pinned_map": {str(k): v for k, v in (pinned or {}).items()}, "steps": steps})
    return cases


def engine_cases():
    """Small simulated SUN runs; record the router's view and the step schedule."""
    out = []
    specs = [
        dict(n_models=4, pool=2, alpha=0.0, rps=4.0, isl=512, osl=64, rule=DecodeRule.LEAST_OUTSTANDING_TOKENS),
        dict(n_models=4, pool=2, alpha=1.5, rps=6.0, isl=1024, osl=32, rule=DecodeRule.LEAST_OUTSTANDING_TOKENS),
        dict(n_models=8, pool=4, alpha=3.0, rps=8.0, isl=256, osl=16, rule=DecodeRule.ROUND_ROBIN),
        dict(n_models=4, pool=3, alpha=1.5, rps=5.0, isl=384, osl=24, rule=DecodeRule.WEIGHTED_RANDOM),
        dict(n_models=4, pool=4, alpha=1.5, rps=5.0, isl=384, osl=24, rule=DecodeRule.PINNED),
    ]
    for sp in specs:
        mode = PoolMode.ISOLATED if sp["rule"] is DecodeRule.PINNED else PoolMode.SHARED
        models = tuple(ModelProfile(model_id=i, param_count=8.03e9, kv_bytes_per_token=131072,
                                    shared_decoder=mode is PoolMode.SHARED) for i in range(sp["n_models"]))
        cluster = ClusterConfig(models=models, decode_pool_mode=mode, decode_pool_size=sp["pool"],
                                routing_policy=RoutingPolicy(decode_rule=sp["rule"], seed=3), gpu_spec=SIMPLE_GPU)
        ws = WorkloadSpec(n_models=sp["n_models"], total_rps=sp["rps"], alpha=sp["alpha"], isl=sp["isl"],
                          osl=sp["osl"], grace_period=1.0, measurement_window=4.0, seed=42)
        trace = generate_trace(ws)
        seen = []
        orig = routing.DecodeDispatcher.route

        def spy(self, request, pool, _orig=orig):
            pick = _orig(self, request, pool)
            seen.append({"request": [request.id, request.model_id], "pool": [snap_dict(s) for s in pool],
                         "pick": pick})
            return pick

        routing.DecodeDispatcher.route = spy
        try:
            res = engine.run(cluster, trace, SIMPLE_COST, record_events=True)
        finally:
            routing.DecodeDispatcher.route = orig
        log = res.resource_log
        out.append({
            "spec": {k: (v.value if hasattr(v, "value") else v) for k, v in sp.items()},
            "policy_seed": 3,
            "router_view": seen,
            "dispatches": log.dispatches,
            "steps": [[w, b, kvb] for (w, _t, _d, b, kvb) in log.steps],
            "charged_steps": log.charged_steps,
            "n_requests": len(trace),
            "events": [[round(t * 1e9), k.name, rid, wid] for (t, k, rid, wid) in res.event_trace],
            "summary": metrics.summarize(measurement_filter(res.completed, ws), cluster, ws).to_dict(),
        })
    return out


def costmodel_values():
    m16 = ModelProfile(model_id=0, param_count=8.03e9)
    m4 = ModelProfile(model_id=1, param_count=8.03e9, decode_weight_bits=4)
    vals = []
    for batch in ([(m16, 1024)], [(m16, 1024), (m16, 2000), (m16, 1)], [(m4, 512)] * 5):
        w = batch[0][0].weight_bytes(poolsim.WorkerRole.DECODE)
        vals.append({"batch": [[m.model_id, m.decode_weight_bits, t] for m, t in batch],
                     "step_time": decode_step_time(batch, w, SIMPLE_COST, SIMPLE_GPU)})
    tr = [{"tokens": t, "bpt": b, "time": transfer_time(KvHandle(0, t, b), SIMPLE_GPU)}
          for t, b in ((1, 131072), (1024, 131072), (16384, 196608))]
    tp = [{"isl": i, "osl": o, "bits": m.decode_weight_bits, "tpot": single_request_tpot(m, i, o, SIMPLE_COST, SIMPLE_GPU)}
          for m in (m16, m4) for i, o in ((1024, 8), (512, 256))]
    # calibrate() on the shipped A100 targets (pkg/configs/targets_llama8b.csv) and on a
    # subset it cannot fit (CalibrationInfeasible); the CSV text travels in the fixture
    from poolsim.costmodel import CalibrationInfeasible, calibrate, load_targets_csv
    csv_path = "/root/reference/pkg/configs/targets_llama8b.csv"
    targets = load_targets_csv(csv_path, 8.03e9, 131072)
    cal = {"csv": open(csv_path).read(), "param_count": 8.03e9, "kv_bytes_per_token": 131072,
           "params": calibrate(targets, GpuSpec()).to_dict()}
    try:
        calibrate(targets, GpuSpec(), rel_tol=0.001)
    except CalibrationInfeasible as e:
        cal["tight_error"] = str(e)
    return {"decode_step_time": vals, "transfer_time": tr, "single_request_tpot": tp, "calibrate": cal}


def workload_values():
    z = [{"n": n, "alpha": a, "total": t, "rates": zipf_split(n, a, t)}
         for n, a, t in ((4, 1.5, 1.0), (8, 1.5, 16.0), (8, 3.0, 2.0), (16, 0.0, 3.5), (1, 2.7, 3.5))]
    traces = []
    for spec in (WorkloadSpec(n_models=4, total_rps=2.0, alpha=0.0, isl=128, osl=16, grace_period=2.0,
                              measurement_window=4.0, drain_margin=0.0, seed=42,
                              arrival_process=ArrivalProcess.DETERMINISTIC),
                 WorkloadSpec(n_models=8, total_rps=10.0, alpha=1.5, isl=1024, osl=256, grace_period=1.0,
                              measurement_window=5.0, seed=42),
                 WorkloadSpec(n_models=16, total_rps=20.0, alpha=3.0, isl=512, osl=64, grace_period=0.5,
                              measurement_window=3.0, seed=7)):
        buf = io.StringIO()
        write_trace(generate_trace(spec), buf)
        traces.append({"spec": {k: (v.value if hasattr(v, "value") else v) for k, v in spec.__dict__.items()},
                       "text": buf.getvalue()})
    return {"zipf": z, "traces": traces}


def cluster_values():
    cases = []
    bad = [
        ClusterConfig(models=(), decode_pool_mode=PoolMode.SHARED, decode_pool_size=0),
        ClusterConfig(models=(ModelProfile(0, 8e9, shared_decoder=True), ModelProfile(0, 7e9, decode_weight_bits=4,
                                                                                     shared_decoder=True)),
                      decode_pool_mode=PoolMode.SHARED, decode_pool_size=2,
                      routing_policy=RoutingPolicy(decode_rule=DecodeRule.PINNED)),
        ClusterConfig(models=(ModelProfile(0, 8e9), ModelProfile(1, 8e9, prefill_weight_bits=8)),
                      decode_pool_mode=PoolMode.ISOLATED, decode_pool_size=3),
        ClusterConfig(models=(ModelProfile(0, 8e11, shared_decoder=True),), decode_pool_mode=PoolMode.SHARED,
                      decode_pool_size=1, gpu_spec=GpuSpec(hbm_bandwidth=-1.0)),
    ]
    for i, c in enumerate(bad):
        try:
            validate_cluster(c)
            cases.append({"case": i, "violations": []})
        except InvalidConfig as e:
            cases.append({"case": i, "violations": e.violations})
    return cases


def main():
    with open(os.path.join(OUT, "router_golden.json"), "w") as f:
        json.dump(router_cases(), f)
    with open(os.path.join(OUT, "engine_golden.json"), "w") as f:
        json.dump({"runs": engine_cases(), "costmodel": costmodel_values()}, f)
    with open(os.path.join(OUT, "workload_golden.json"), "w") as f:
        json.dump(workload_values(), f)
    with open(os.path.join(OUT, "cluster_golden.json"), "w") as f:
        json.dump(cluster_values(), f, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
