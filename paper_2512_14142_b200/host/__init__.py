"""Host side of the data path: the reference's plugin API, restated.

The names, argument meanings and error behaviour follow the reference's
public surface (reference: pkg/src/agentsched/__init__.py:12-140) for the
parts the GPU data path sits behind: traces, cost tables, scheduling
policies, the KV policy + memory model, the event loop and the report.
"""

from .costs import (ApiLatencyTable, DecodeModel, PrefillProfile, ServiceTimePredictor,
                    figure2_predictor)
from .engine import (COST_MODELS, DEFAULT_CAPACITY_TOKENS, PARALLEL_MAX, SERIAL,
                     AdmittedMember, Engine, EventKind, SimConfig, execute_batch, run)
from .errors import (ConfigError, DeviceError, ProtocolError, SimulationError,
                     TraceParseError, ValidationError)
from .kvpolicy import (ACTION_PREFERENCE, CacheAction, KvCacheManager, MemoryModel,
                       WasteEstimate, audit_conservation, estimate_waste)
from .policies import (POLICIES, BatchPlan, CacheLocation, FcfsPolicy, LasPolicy, MlfqConfig,
                       Phase, RequestSjfPolicy, RequestState, SchedulingPolicy, SegmentSjfPolicy,
                       StatefulMlfqPolicy, hrrn_score, kv_demand, make_policy)
from .report import (GanttSpan, RequestRecord, RunReport, audit_time_decomposition,
                     audit_waste_log, avg_jct, degradation_ratio, percentile)
from .trace import (ApiCategory, LatencySpec, RequestSpec, SegmentSpec, TokenRange,
                    WorkloadConfig, figure2_workload, generate, load_trace, save_trace,
                    segment_token_ids, workload_hash)

__all__ = [n for n in dir() if not n.startswith("_")]
