"""bench.py's multi-GPU request placement (CPU): the reference router (LOT,
anticipatory load) spreads the Zipf-skewed C3 trace evenly over N decode
workers with every model on every worker (weak scaling, no collective on the
data path); PINNED (the per-model partitioned baseline) maps model i -> worker
i mod N."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lot_spreads_the_zipf_mix_evenly(world):
    per = bench.build_assignment(bench.CONFIGS["c3"], world, "lot")
    assert [len(p) for p in per] == [64] * world
    ids = [r for p in per for r, _ in p]
    assert len(ids) == len(set(ids)) == 64 * world
    if world <= 4:  # every GPU decodes a mix of task models (model-agnostic shared decode)
        assert all(len({m for _, m in p}) >= 4 for p in per)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_pinned_is_model_partitioned(world):
    per = bench.build_assignment(bench.CONFIGS["c3"], world, "pinned")
    for w, p in enumerate(per):
        assert {m % world for _, m in p} <= {w}
    sizes = [len(p) for p in per]
    assert sum(sizes) == 64 * world and sizes[0] == max(sizes)  # Zipf: model 0's worker is the hot one
