"""bench.py's N-rank path on CPU (gloo, world size 2): `--gpus 2` outside torchrun
spawns the ranks itself, the ranks route the Zipf trace with the reference
router, time with a barrier + max-over-ranks all-reduce, and rank 0 prints one
JSON line; on a box with fewer GPUs than asked the GPU arm fails loudly."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_spawns_two_ranks_and_aggregates():
    import bench

    r = _run(["--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["dry_run"]
    assert line["config"]["global_batch"] == 2 * 64 and line["config"]["batch_per_gpu"] == 64
    # the same LOT routing the GPU arm uses: both workers hold a mix of task models
    want = [sorted({m for _, m in w}) for w in bench.build_assignment(bench.CONFIGS["c3"], 2, "lot")]
    assert line["config"]["models_per_rank"] == want
    assert abs(line["value"] - 2 * 64 * 3 / (line["ms_per_step"] * 3 / 1e3)) < 1e-6 * line["value"]


def test_bench_pinned_routing_partitions_models():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "3", "--routing", "pinned"])
    assert r.returncode == 0, r.stderr[-2000:]
    per = _line(r.stdout)["config"]["models_per_rank"]
    assert per == [[0, 2, 4, 6], [1, 3, 5, 7]]  # PINNED: model i -> worker i mod 2


def test_bench_refuses_more_gpus_than_visible():
    import torch

    if torch.cuda.device_count() >= 2:
        return
    r = _run(["--gpus", "2", "--steps", "3"])
    assert r.returncode != 0 and "CUDA device" in (r.stderr + r.stdout)
