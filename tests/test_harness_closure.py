"""Harness closure: the reference's decode cost model refit to
B200-measured step times (tests/golden/b200_steps_8b_*.json, made on a B200 by
scripts/measure_step_grid.py), and the measured-table backend that lets the
reference-semantics serving loop predict the B200 system."""
import json
import os

import pytest

from paper_2603_02599_b200 import pricing, scheduler
from paper_2603_02599_b200.errors import CalibrationInfeasible
from paper_2603_02599_b200.sun_types import DecodeRule, GpuSpec, Request

from .test_scheduler import COST, cluster

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = GpuSpec.b200(6463.3, 1666.0)


def _load(name):
    return pricing.load_step_points(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("name", ["b200_steps_8b_bf16.json", "b200_steps_8b_w4.json"])
def test_reference_form_refit_and_its_limit(name):
    hdr, pts = _load(name)
    # the reference's affine form (D + bytes / (mbu * BW)) fits the B200 only loosely:
    # GEMM time grows with the batch (tensor work, activation traffic), bytes do not say so
    d, mbu, res = pricing.calibrate_decode(pts, hdr["decode_weight_bytes"], hdr["kv_bytes_per_token"], B200,
                                           rel_tol=0.35)
    assert 0.0 < d < 5e-3 and 0.5 < mbu <= 1.0
    assert len(res) == len(pts)
    with pytest.raises(CalibrationInfeasible) as e:  # the reference's 3% tolerance is out of reach
        pricing.calibrate_decode(pts, hdr["decode_weight_bytes"], hdr["kv_bytes_per_token"], B200)
    errs = [abs(x) for _, x in e.value.residuals]
    assert errs == sorted(errs, reverse=True) and errs[0] > 0.03


def test_calibrate_decode_rejects_like_the_reference():
    with pytest.raises(CalibrationInfeasible):
        pricing.calibrate_decode([pricing.StepPoint(1, 1024, 1e-3)], 1e9, 1e5, B200)
    # faster than the HBM allows -> mbu > 1
    pts = [pricing.StepPoint(1, c, 1e-6 + c * 1e5 / 1e14) for c in (256, 1024, 4096)]
    with pytest.raises(CalibrationInfeasible):
        pricing.calibrate_decode(pts, 0.0, 1e5, B200)


@pytest.mark.parametrize("name", ["b200_steps_8b_bf16.json", "b200_steps_8b_w4.json"])
def test_measured_backend_exact_on_grid_and_monotone(name):
    hdr, pts = _load(name)
    mb = pricing.MeasuredBackend(pts, hdr["kv_bytes_per_token"])
    for p in pts:
        assert mb.predict(p.batch, p.context) == pytest.approx(p.step_s, rel=1e-12)
        kv = p.batch * p.context * hdr["kv_bytes_per_token"]
        assert mb.step_time(kv, hdr["decode_weight_bytes"], p.batch) == pytest.approx(p.step_s, rel=1e-12)
    for b in (1, 24, 64, 100):
        ts = [mb.predict(b, c) for c in (100, 256, 700, 1500, 3000, 4096, 6000)]
        assert ts == sorted(ts)
    for c in (300, 1100, 5000):
        ts = [mb.predict(b, c) for b in (1, 5, 16, 40, 64, 128)]
        assert ts == sorted(ts)
    with pytest.raises(ValueError):
        mb.step_time(1e9, 1e9)


def test_measured_backend_predicts_the_c3_bench():
    """The grid (equal contexts) predicts the C3 bench step (64 mixed members,
    contexts 1024..1279 growing while timed) within 3%."""
    hdr, pts = _load("b200_steps_8b_bf16.json")
    mb = pricing.MeasuredBackend(pts, hdr["kv_bytes_per_token"])
    line = json.load(open(os.path.join(ROOT, "profiles", "r02", "bench_c3_n1.json")))
    ctx_mean = (line["config"]["ctx_min"] + line["config"]["ctx_max"]) / 2 + line["warmup"] + line["steps"] / 2
    pred = mb.predict(line["config"]["batch_per_gpu"], ctx_mean)
    assert pred == pytest.approx(line["ms_per_step"] / 1e3, rel=0.03)


def test_serving_loop_on_measured_b200_steps():
    """The reference-semantics serving loop priced by the B200 table: every
    logged step duration is the table's price for that batch and KV."""
    hdr, pts = _load("b200_steps_8b_bf16.json")
    mb = pricing.MeasuredBackend(pts, hdr["kv_bytes_per_token"])
    cfg = cluster(4, 1, DecodeRule.LEAST_OUTSTANDING_TOKENS, gpu=B200)
    trace = [Request(id=i, model_id=i % 4, arrival_time=0.001 * i, isl=1024, target_osl=16) for i in range(48)]
    res = scheduler.run(cfg, trace, COST, backend=mb)
    assert len(res.completed) == 48
    for (_w, _t, dur, b, kvb) in res.log.steps:
        assert dur == pytest.approx(mb.step_time(kvb, 0.0, b), rel=1e-12)
    # the analytic reference price differs (it has no batch term)
    ana = scheduler.run(cfg, trace, COST)
    assert [s[2] for s in ana.log.steps] != [s[2] for s in res.log.steps]


# poolsim harness.py:33-45 ROW_FIELDS (the reference's row schema, as its module builds it)
REFERENCE_ROW_FIELDS = [
    "config_hash", "decode_pool_mode", "decode_pool_size", "alpha", "isl", "osl", "offered_rps",
    "completed_requests", "ttft_mean_s", "ttft_p50_s", "ttft_p99_s", "tpot_mean_s", "tpot_p50_s", "tpot_p99_s",
    "itl_mean_s", "interactivity_tok_s", "output_throughput_tok_s", "throughput_per_decode_gpu_tok_s",
    "throughput_per_gpu_all_tok_s", "achieved_rps", "achieved_offered_ratio", "seed", "cell_index", "replicate",
    "error"]
ROWS_CSV = os.path.join(GOLDEN, "b200_consolidation_rows.csv")


def test_row_schema_is_the_reference_one():
    import csv
    import subprocess
    import sys

    from paper_2603_02599_b200 import harness

    assert harness.ROW_FIELDS == REFERENCE_ROW_FIELDS
    with open(ROWS_CSV) as fh:
        assert next(csv.reader(fh)) == REFERENCE_ROW_FIELDS
    src = "/root/reference/pkg/src"
    if os.path.isdir(src):  # the build container: check against the reference module itself
        out = subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r); "
                              "from poolsim.harness import ROW_FIELDS; print(','.join(ROW_FIELDS))" % src],
                             capture_output=True, text=True, cwd="/tmp", env={**os.environ,
                                                                               "PYTHONDONTWRITEBYTECODE": "1"})
        assert out.returncode == 0, out.stderr
        assert out.stdout.strip().split(",") == REFERENCE_ROW_FIELDS


def test_consolidation_rows_reproduce_and_shared_tpot_within_5pct():
    """The committed rows (scripts/harness_rows.py: sweep_consolidation.toml's axes plus the
    4 x 1P/1D partition, decode priced by the B200 step table) are reproduced exactly, and
    the shared pool's TPOT p50 is within 5% of (here: at or below) the per-model partition's
    at equal GPU count (north star: TPOT within 5% of a partitioned decode)."""
    import csv
    import io

    from paper_2603_02599_b200 import harness
    from scripts.harness_rows import COST

    hdr, pts = _load("b200_steps_8b_bf16.json")
    backend = pricing.MeasuredBackend(pts, hdr["kv_bytes_per_token"])
    cells = harness.consolidation_cells(B200)[:5]  # alpha 0, osl 128: the partition + pools 4..1
    rows = [harness.run_cell(c, COST, backend, "b200-measured:b200_steps_8b_bf16.json") for c in cells]
    buf = io.StringIO()
    harness.write_rows(rows, buf)
    committed = open(ROWS_CSV).read().splitlines()
    assert buf.getvalue().splitlines() == committed[:6]
    table = list(csv.DictReader(open(ROWS_CSV)))
    assert len(table) == 20 and not any(r["error"] for r in table)
    for (alpha, osl) in [("0.0", "128"), ("0.0", "256"), ("1.5", "128"), ("1.5", "256")]:
        sel = [r for r in table if r["alpha"] == alpha and r["osl"] == osl]
        iso = [r for r in sel if r["decode_pool_mode"] == "isolated"][0]
        sh4 = [r for r in sel if r["decode_pool_mode"] == "shared" and r["decode_pool_size"] == "4"][0]
        assert float(sh4["tpot_p50_s"]) <= 1.05 * float(iso["tpot_p50_s"])
        # consolidation: per-decode-GPU throughput grows as the shared pool shrinks
        thr = [float(r["throughput_per_decode_gpu_tok_s"]) for r in sel if r["decode_pool_mode"] == "shared"]
        assert thr == sorted(thr)
