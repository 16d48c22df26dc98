"""Harness closure: the reference's experiment rows, produced by
the reference-semantics serving loop priced by the real B200 decode step.

poolsim's harness (pkg/src/poolsim/harness.py:33-45, 141-169) turns one run into a
row of ``ROW_FIELDS``: cluster / workload identity, the ``RunSummary`` of the
measurement window (metrics.py:102-150) and the sweep coordinates. Here the same
rows come from ``scheduler.run`` — the restated engine — with the decode step
priced by ``pricing.MeasuredBackend``, i.e. the step times measured on a B200 by
``scripts/measure_step_grid.py`` (tests/golden/b200_steps_8b_*.json), at the
engine.py:427 call site. The sweep/TOML layer itself is out of scope;
``consolidation_cells`` restates configs/sweep_consolidation.toml's axes over the
B200 so the consolidation question (shared pool vs per-model partition, PAPER.md
§6) is answered with the real step.

``config_hash`` is a sha256 prefix of the run's canonical JSON like poolsim's
(config.py:349-351), over this package's dataclasses (poolsim hashes its TOML
layout, config_to_dict, which is out of scope): identical inputs give identical
hashes, not poolsim's strings.
"""
from __future__ import annotations

import csv
import dataclasses
import hashlib
import json
from dataclasses import dataclass
from enum import Enum
from typing import IO, Iterable

from . import pricing, scheduler
from .errors import InvalidConfig
from .stats import EmptyWindow, IncompleteRequest, RunSummary, summarize
from .sun_types import ClusterConfig, DecodeRule, GpuSpec, ModelProfile, PoolMode, RoutingPolicy
from .trace import WorkloadSpec, generate_trace, measurement_filter

# metrics.py SUMMARY_FIELDS (RunSummary's field order)
SUMMARY_FIELDS = [f.name for f in dataclasses.fields(RunSummary)]

# harness.py:33-45
ROW_FIELDS = (
    ["config_hash", "decode_pool_mode", "decode_pool_size", "alpha", "isl", "osl", "offered_rps"]
    + [f for f in SUMMARY_FIELDS if f != "offered_rps"]
    + ["seed", "cell_index", "replicate", "error"]
)


def _canon(x):
    if dataclasses.is_dataclass(x):
        return {f.name: _canon(getattr(x, f.name)) for f in dataclasses.fields(x)}
    if isinstance(x, Enum):
        return x.value
    if isinstance(x, (list, tuple)):
        return [_canon(v) for v in x]
    return x


def config_hash(cluster: ClusterConfig, workload: WorkloadSpec, cost: pricing.CostParams, backend: str) -> str:
    canonical = json.dumps({"cluster": _canon(cluster), "workload": _canon(workload), "cost": _canon(cost),
                            "decode_backend": backend}, sort_keys=True)
    return hashlib.sha256(canonical.encode()).hexdigest()[:12]


def summary_row(cluster: ClusterConfig, workload: WorkloadSpec, chash: str, summary: RunSummary | None,
                error: str = "", cell_index: int = 0, replicate: int = 0) -> dict:
    """harness.py:141-169 summary_row: one result row from a summary (or an error)."""
    row = {"config_hash": chash, "decode_pool_mode": cluster.decode_pool_mode.value,
           "decode_pool_size": cluster.decode_pool_size, "alpha": workload.alpha, "isl": workload.isl,
           "osl": workload.osl, "offered_rps": workload.total_rps, "seed": workload.seed, "cell_index": cell_index,
           "replicate": replicate, "error": error}
    sd = summary.to_dict() if summary is not None else {}
    for name in SUMMARY_FIELDS:
        if name != "offered_rps":
            row[name] = sd.get(name, "")
    return row


@dataclass(frozen=True)
class Cell:
    index: int
    replicate: int
    cluster: ClusterConfig
    workload: WorkloadSpec


def run_cell(cell: Cell, cost: pricing.CostParams, backend: pricing.DecodeBackend, backend_name: str) -> dict:
    """One run end to end (harness.py run_single + summary_row); a failing cell becomes
    a row with its error column set (harness.py _cell_row)."""
    chash = config_hash(cell.cluster, cell.workload, cost, backend_name)
    try:
        trace = generate_trace(cell.workload)
        res = scheduler.run(cell.cluster, trace, cost, horizon=cell.workload.horizon, backend=backend)
        summary = summarize(measurement_filter(res.completed, cell.workload), cell.cluster, cell.workload)
        return summary_row(cell.cluster, cell.workload, chash, summary, "", cell.index, cell.replicate)
    except (InvalidConfig, EmptyWindow, IncompleteRequest, scheduler.SimulationDiverged) as e:
        return summary_row(cell.cluster, cell.workload, chash, None, f"{type(e).__name__}: {e}", cell.index,
                           cell.replicate)


def write_rows(rows: Iterable[dict], fh: IO[str]) -> None:
    w = csv.DictWriter(fh, fieldnames=ROW_FIELDS, lineterminator="\n")
    w.writeheader()
    for r in rows:
        w.writerow({k: (repr(v) if isinstance(v, float) else v) for k, v in r.items()})


def b200_cluster(n_models: int, pool: int, shared: bool, gpu: GpuSpec, param_count: float = 8.03e9,
                 kv_bytes_per_token: int = 131072, decode_bits: int = 16, seed: int = 0) -> ClusterConfig:
    """configs/cluster_shared.toml / cluster_baseline.toml on B200s: n task models on
    dedicated prefill GPUs, a shared least-outstanding-tokens pool or per-model pinned
    decode workers."""
    mode = PoolMode.SHARED if shared else PoolMode.ISOLATED
    rule = DecodeRule.LEAST_OUTSTANDING_TOKENS if shared else DecodeRule.PINNED
    models = tuple(ModelProfile(model_id=i, param_count=param_count, kv_bytes_per_token=kv_bytes_per_token,
                                decode_weight_bits=decode_bits, shared_decoder=shared) for i in range(n_models))
    return ClusterConfig(models=models, decode_pool_mode=mode, decode_pool_size=pool,
                         routing_policy=RoutingPolicy(decode_rule=rule, seed=seed), gpu_spec=gpu)


def consolidation_cells(gpu: GpuSpec, rps: float = 24.0, alphas=(0.0, 1.5), osls=(128, 256),
                        pools=(4, 3, 2, 1), n_models: int = 4, isl: int = 1024, window: float = 20.0,
                        grace: float = 5.0, seed: int = 42) -> list[Cell]:
    """configs/sweep_consolidation.toml's axes (offered_rps, decode_pool_size, alpha, osl)
    over cluster_shared.toml, plus the cluster_baseline.toml partition (4 x 1P/1D,
    pinned) at each (alpha, osl): the per-model partitioned decode of the same step."""
    cells, idx = [], 0
    for alpha in alphas:
        for osl in osls:
            wl = WorkloadSpec(n_models=n_models, total_rps=rps, alpha=alpha, isl=isl, osl=osl, grace_period=grace,
                              measurement_window=window, seed=seed)
            cells.append(Cell(idx, 0, b200_cluster(n_models, n_models, False, gpu), wl))
            idx += 1
            for pool in pools:
                cells.append(Cell(idx, 0, b200_cluster(n_models, pool, True, gpu), wl))
                idx += 1
    return cells


__all__ = ["Cell", "ROW_FIELDS", "SUMMARY_FIELDS", "b200_cluster", "config_hash", "consolidation_cells", "run_cell",
           "summary_row", "write_rows"]
