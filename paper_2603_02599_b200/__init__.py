"""B200-native SUN shared decode path (arxiv 2603.02599).

The reference (poolsim) API names are re-exported so code written against it
keeps working; the decode step itself runs in libsun_b200.so (sm_100a).
"""
from .errors import (EmptyPool, InvalidConfig, MixedDecoderError, OverCapacity, SunCudaError, UnknownModel,
                     UnsupportedShape)
from .pricing import (AnalyticBackend, CostParams, DecodeBackend, decode_step_time, decode_step_time_from_totals,
                      kv_step_bytes, single_request_tpot, step_bytes, transfer_time)
from .router import DecodeDispatcher, PoolSnapshot, outstanding_tokens, route_prefill
from .spec import LLAMA31_8B, LLAMA32_1B, QWEN25_14B, SPECS, TINY, DecoderSpec
from .stats import EmptyWindow, IncompleteRequest, RunSummary, nearest_rank, per_request_metrics, summarize
from .sun_types import (IN_TRANSIT, ClusterConfig, DecodeRule, GpuSpec, KvHandle, ModelProfile, PoolMode, Request,
                        RequestOutcome, RoutingPolicy, WorkerRole, WorkerState, decode_worker_ids,
                        pinned_decode_worker, prefill_worker_id, validate_cluster)
from .trace import (ArrivalProcess, WorkloadSpec, generate_trace, measurement_filter, read_trace, write_trace,
                    zipf_split)

__version__ = "0.1.0"
