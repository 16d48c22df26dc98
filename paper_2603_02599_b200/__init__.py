"""B200-native SUN shared decode path (arxiv 2603.02599).

The reference (poolsim) API names are re-exported so code written against it
keeps working; the decode step itself runs in libsun_b200.so (sm_100a).
"""
from .errors import (CalibrationInfeasible, EmptyPool, InvalidConfig, MixedDecoderError, OverCapacity, SunCudaError,
                     UnknownModel, UnsupportedShape)
from .pricing import (AnalyticBackend, CalibrationTarget, CostParams, DecodeBackend, MeasuredBackend, calibrate,
                      calibrate_decode, decode_step_time, decode_step_time_from_totals, kv_step_bytes,
                      load_targets_csv, prefill_time, single_request_tpot, single_request_ttft, step_bytes,
                      transfer_time)
from .harness import ROW_FIELDS, SUMMARY_FIELDS, summary_row
from .scheduler import SimResult, SimulationDiverged, run
from .router import DecodeDispatcher, PoolSnapshot, outstanding_tokens, route_prefill
from .spec import LLAMA31_8B, LLAMA32_1B, QWEN25_14B, SPECS, TINY, DecoderSpec
from .stats import EmptyWindow, IncompleteRequest, RunSummary, nearest_rank, per_request_metrics, summarize
from .sun_types import (IN_TRANSIT, ClusterConfig, DecodeRule, GpuSpec, KvHandle, ModelProfile, PoolMode, Request,
                        RequestOutcome, RoutingPolicy, WorkerRole, WorkerState, decode_worker_ids,
                        pinned_decode_worker, prefill_worker_id, validate_cluster)
from .trace import (ArrivalProcess, WorkloadSpec, generate_trace, measurement_filter, read_trace, write_trace,
                    zipf_split)

__version__ = "0.2.0"

# poolsim.__all__ (pkg/src/poolsim/__init__.py:49-94) minus its config / sweep /
# CLI names (RunConfig, SweepSpec, load_config, run_single, run_sweep: SURVEY §2
# out of scope), plus the B200 path's own names
__all__ = [
    "ArrivalProcess", "CalibrationInfeasible", "CalibrationTarget", "ClusterConfig", "CostParams",
    "DecodeDispatcher", "DecodeRule", "EmptyPool", "EmptyWindow", "GpuSpec", "IncompleteRequest", "InvalidConfig",
    "KvHandle", "MixedDecoderError", "ModelProfile", "PoolMode", "PoolSnapshot", "Request", "RequestOutcome",
    "RoutingPolicy", "RunSummary", "SimResult", "SimulationDiverged", "UnknownModel", "WorkerRole", "WorkerState",
    "WorkloadSpec", "calibrate", "decode_step_time", "generate_trace", "measurement_filter", "per_request_metrics",
    "prefill_time", "route_prefill", "run", "summarize", "transfer_time", "validate_cluster", "zipf_split",
    # B200 path
    "AnalyticBackend", "DecodeBackend", "MeasuredBackend", "OverCapacity", "SunCudaError", "UnsupportedShape",
    "DecoderSpec", "SPECS", "TINY", "LLAMA32_1B", "LLAMA31_8B", "QWEN25_14B", "calibrate_decode",
    "decode_step_time_from_totals", "kv_step_bytes", "load_targets_csv", "nearest_rank", "outstanding_tokens",
    "single_request_tpot", "single_request_ttft", "step_bytes", "read_trace", "write_trace",
    "ROW_FIELDS", "SUMMARY_FIELDS", "summary_row",
]
