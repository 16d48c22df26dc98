"""Host-side mirror of the reference API (types, invariants, pricing, traces,
metrics) against reference golden values (tests/golden/, made by
make_golden.py from /root/reference/pkg/src/poolsim)."""
import io
import json
import os

import pytest

import paper_2603_02599_b200 as sun
from paper_2603_02599_b200 import pricing, stats, trace
from paper_2603_02599_b200.errors import InvalidConfig, MixedDecoderError
from paper_2603_02599_b200.sun_types import (ClusterConfig, DecodeRule, GpuSpec, KvHandle, ModelProfile, PoolMode,
                                             Request, RoutingPolicy, WorkerRole, validate_cluster)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SIMPLE_COST = pricing.CostParams(prefill_flops_per_token=2.0e10, prefill_fixed_overhead=0.01,
                                 decode_fixed_overhead=0.002, dequant_compute_penalty=1.25, mfu=0.5, mbu=0.8)
SIMPLE_GPU = GpuSpec(flops=1.0e14, hbm_bandwidth=1.0e12, hbm_capacity=8.0e10, interconnect_bandwidth=5.0e10,
                     interconnect_latency=1.0e-4)


def test_public_names_match_reference_surface():
    for name in ("KvHandle", "ModelProfile", "DecodeDispatcher", "PoolSnapshot", "RoutingPolicy", "DecodeRule",
                 "route_prefill", "decode_step_time", "MixedDecoderError", "validate_cluster", "zipf_split",
                 "generate_trace", "summarize", "transfer_time", "GpuSpec", "ClusterConfig", "Request"):
        assert hasattr(sun, name), name


def test_costmodel_values_match_reference():
    g = json.load(open(os.path.join(GOLDEN, "engine_golden.json")))["costmodel"]
    for case in g["decode_step_time"]:
        batch = [(ModelProfile(model_id=mid, param_count=8.03e9, decode_weight_bits=bits), t)
                 for mid, bits, t in case["batch"]]
        w = batch[0][0].weight_bytes(WorkerRole.DECODE)
        assert pricing.decode_step_time(batch, w, SIMPLE_COST, SIMPLE_GPU) == case["step_time"]
    for case in g["transfer_time"]:
        assert pricing.transfer_time(KvHandle(0, case["tokens"], case["bpt"]), SIMPLE_GPU) == case["time"]
    for case in g["single_request_tpot"]:
        m = ModelProfile(model_id=0, param_count=8.03e9, decode_weight_bits=case["bits"])
        assert pricing.single_request_tpot(m, case["isl"], case["osl"], SIMPLE_COST, SIMPLE_GPU) == case["tpot"]


def test_calibrate_matches_reference(tmp_path):
    """pricing.calibrate on the reference's shipped A100 targets gives the reference's
    CostParams exactly (costmodel.py:257-358; the A100 constants of
    cluster_shared.toml:38-44), and a tolerance it cannot meet raises
    CalibrationInfeasible with the same residual report."""
    import paper_2603_02599_b200 as sun

    g = json.load(open(os.path.join(GOLDEN, "engine_golden.json")))["costmodel"]["calibrate"]
    path = tmp_path / "targets.csv"
    path.write_text(g["csv"])
    targets = sun.load_targets_csv(str(path), g["param_count"], g["kv_bytes_per_token"])
    params = sun.calibrate(targets, sun.GpuSpec())
    assert params.to_dict() == g["params"]
    with pytest.raises(sun.CalibrationInfeasible) as ei:
        sun.calibrate(targets, sun.GpuSpec(), rel_tol=0.001)
    assert str(ei.value) == g["tight_error"]
    with pytest.raises(sun.CalibrationInfeasible):
        sun.calibrate(targets[:1], sun.GpuSpec())


def test_package_root_names_cover_reference_api():
    """poolsim.__all__ (pkg/src/poolsim/__init__.py:49-94) minus the out-of-scope
    config / sweep names is importable from the package root."""
    import paper_2603_02599_b200 as sun

    ref_all = ["ArrivalProcess", "CalibrationInfeasible", "CalibrationTarget", "ClusterConfig", "CostParams",
               "DecodeDispatcher", "DecodeRule", "EmptyPool", "EmptyWindow", "GpuSpec", "IncompleteRequest",
               "InvalidConfig", "KvHandle", "MixedDecoderError", "ModelProfile", "PoolMode", "PoolSnapshot", "Request",
               "RequestOutcome", "RoutingPolicy", "RunConfig", "RunSummary", "SimResult", "SimulationDiverged",
               "SweepSpec", "UnknownModel", "WorkerRole", "WorkerState", "WorkloadSpec", "calibrate",
               "decode_step_time", "generate_trace", "load_config", "measurement_filter", "per_request_metrics",
               "prefill_time", "route_prefill", "run", "run_single", "run_sweep", "summarize", "transfer_time",
               "validate_cluster", "zipf_split"]
    out_of_scope = {"RunConfig", "SweepSpec", "load_config", "run_single", "run_sweep"}
    for name in ref_all:
        if name not in out_of_scope:
            assert name in sun.__all__ and hasattr(sun, name), name


def test_decode_step_time_errors_like_reference():
    a = ModelProfile(0, 8.03e9)
    b = ModelProfile(1, 8.03e9, decode_weight_bits=4)
    with pytest.raises(MixedDecoderError):
        pricing.decode_step_time([(a, 10), (b, 10)], 1.0, SIMPLE_COST, SIMPLE_GPU)
    with pytest.raises(ValueError):
        pricing.decode_step_time([], 1.0, SIMPLE_COST, SIMPLE_GPU)
    with pytest.raises(ValueError):
        pricing.transfer_time(KvHandle(0, 0, 131072), SIMPLE_GPU)
    # amortisation: weights charged once per step (pkg/tests/test_costmodel.py:74-80)
    w = a.weight_bytes(WorkerRole.DECODE)
    one = pricing.decode_step_time([(a, 100)], w, SIMPLE_COST, SIMPLE_GPU)
    two = pricing.decode_step_time([(a, 100), (a, 100)], w, SIMPLE_COST, SIMPLE_GPU)
    assert two - one == pytest.approx(100 * 131072 / (0.8 * 1e12), rel=1e-12)


def test_validate_cluster_violations_match_reference():
    cases = json.load(open(os.path.join(GOLDEN, "cluster_golden.json")))
    built = [
        ClusterConfig(models=(), decode_pool_mode=PoolMode.SHARED, decode_pool_size=0),
        ClusterConfig(models=(ModelProfile(0, 8e9, shared_decoder=True),
                              ModelProfile(0, 7e9, decode_weight_bits=4, shared_decoder=True)),
                      decode_pool_mode=PoolMode.SHARED, decode_pool_size=2,
                      routing_policy=RoutingPolicy(decode_rule=DecodeRule.PINNED)),
        ClusterConfig(models=(ModelProfile(0, 8e9), ModelProfile(1, 8e9, prefill_weight_bits=8)),
                      decode_pool_mode=PoolMode.ISOLATED, decode_pool_size=3),
        ClusterConfig(models=(ModelProfile(0, 8e11, shared_decoder=True),), decode_pool_mode=PoolMode.SHARED,
                      decode_pool_size=1, gpu_spec=GpuSpec(hbm_bandwidth=-1.0)),
    ]
    for c, cfg in zip(cases, built):
        try:
            validate_cluster(cfg)
            got = []
        except InvalidConfig as e:
            got = e.violations
        assert got == c["violations"]


def test_zipf_and_traces_byte_identical_to_reference():
    g = json.load(open(os.path.join(GOLDEN, "workload_golden.json")))
    for z in g["zipf"]:
        assert trace.zipf_split(z["n"], z["alpha"], z["total"]) == z["rates"]
    for t in g["traces"]:
        sp = dict(t["spec"])
        sp["arrival_process"] = trace.ArrivalProcess(sp["arrival_process"])
        buf = io.StringIO()
        trace.write_trace(trace.generate_trace(trace.WorkloadSpec(**sp)), buf)
        assert buf.getvalue() == t["text"]
        again = trace.read_trace(io.StringIO(t["text"]))
        buf2 = io.StringIO()
        trace.write_trace(again, buf2)
        assert buf2.getvalue() == t["text"]
    # reference known answer (pkg/tests/test_workload.py:21-31)
    got = trace.zipf_split(4, 1.5, 1.0)
    for g_, e in zip(got, [0.59844, 0.21158, 0.11517, 0.07481]):
        assert g_ == pytest.approx(e, abs=5e-6)


def test_metrics_formulas():
    r = Request(id=0, model_id=0, arrival_time=0.0, isl=8, target_osl=5)
    r.first_token_time, r.completion_time, r.realized_osl = 0.5, 1.3, 5
    ttft, tpot, e2e = stats.per_request_metrics(r)
    assert (ttft, e2e) == (0.5, 1.3) and tpot == pytest.approx(0.2)
    assert stats.nearest_rank([5, 1, 3, 2, 4], 50) == 3
    assert stats.nearest_rank([1, 2, 3, 4], 99) == 4


def test_step_bytes_model():
    from paper_2603_02599_b200.spec import LLAMA31_8B

    sb = pricing.step_bytes(LLAMA31_8B, [1024 + (j * 256) // 64 for j in range(64)])
    assert 24.5e9 < sb < 24.9e9  # C3 = 24.72 GB / step
    assert LLAMA31_8B.kv_bytes_per_token == 131072


def test_step_flags_and_chain_selection():
    """Decode batches (distinct rows) set SUN_STEP_DISTINCT_ROWS and take the bf16 layer
    chain; token-parallel prefill rows do neither; the env switch forces either way and
    (QSUN: up to 128 rows; mirrors sun_capi.cu use_chain)."""
    from paper_2603_02599_b200 import _lib
    from paper_2603_02599_b200.modules import PrefillModule, SharedDecodeModule, uses_gemm_chain

    assert _lib.SUN_STEP_DISTINCT_ROWS == 2 and _lib.SUN_STEP_FEEDBACK == 1
    hdr = open(os.path.join(os.path.dirname(GOLDEN), "..", "include", "sun_b200.h")).read()
    assert "#define SUN_STEP_DISTINCT_ROWS 2" in hdr and "#define SUN_STEP_FEEDBACK 1" in hdr
    assert SharedDecodeModule.distinct_rows and not PrefillModule.distinct_rows
    assert uses_gemm_chain(16, True, None) and not uses_gemm_chain(16, False, None)
    assert uses_gemm_chain(16, False, "1") and not uses_gemm_chain(16, True, "0")
    assert not uses_gemm_chain(16, True, "x") and not uses_gemm_chain(4, True, "0")
    # QSUN: the W4 layer chain up to 128 rows, separate launches above
    assert uses_gemm_chain(4, True, None, batch=128) and not uses_gemm_chain(4, True, None, batch=129)
    assert uses_gemm_chain(4, False, "1", batch=17) and not uses_gemm_chain(4, True, "1", batch=256)
    # QSUN steps of <= 8 rows run the small-batch W4 GEMV (SUN_W4_GEMV=0: the chain / tcgen05 path)
    from paper_2603_02599_b200.modules import uses_w4_gemv

    assert uses_w4_gemv(4, 8, None) and not uses_w4_gemv(4, 9, None) and not uses_w4_gemv(16, 1, None)
    assert not uses_w4_gemv(4, 1, "0") and uses_w4_gemv(4, 1, "1")
    if os.environ.get("SUN_W4_GEMV", "1") != "0" and os.environ.get("SUN_W4_GEMV_CHAIN", "0") == "0":
        assert not uses_gemm_chain(4, True, None, batch=8) and uses_gemm_chain(4, True, None, batch=9)
