"""B200-native multiplicative LLM request router.

Drop-in for the reference ``routesim`` scheduler API on its routing hot path:
the same config dataclasses, ``TraceRecord``, ``ClusterSim`` / ``route`` /
``run_trace`` / ``run`` and ``RunReport``, with every routing decision (chain
hashing, KV$ prefix probe, multiplicative score, rotating-tie-break argmin,
engine + cache state updates) executed by librsim's sm_100a kernels.
"""

from .config import (CacheConfig, CacheFullError, ClusterConfig, CostModel, DetectorConfig, DuplicateRequestError,
                     InvariantError, NoInstancesError, PolicyConfig, UnsupportedConfigError)
from .hashing import chain_keys, combine64, splitmix64, stable_key
from .report import RequestMetrics, RoutingDecision, RunReport, StepRecord, percentile
from .metrics import export, summarize
from .trace import (ClassSpec, PackedTrace, SyntheticSpec, TraceError, TraceRecord, class_key,
                    generate_synthetic, generate_synthetic_packed, load_packed, load_trace, load_trace_packed, save_packed,
                    save_trace, scale_trace)

INFINITE = None


def __getattr__(name):
    # the device-backed entry points import librsim lazily so config/trace
    # tooling works on machines without a GPU
    if name in ("ClusterSim", "run", "probe_capacity", "AdmissionInfo"):
        from . import cluster
        return getattr(cluster, name)
    raise AttributeError(name)


__all__ = [
    "CacheConfig", "CacheFullError", "ClassSpec", "ClusterConfig", "ClusterSim", "CostModel",
    "DetectorConfig", "DuplicateRequestError", "INFINITE", "InvariantError", "NoInstancesError", "PackedTrace",
    "PolicyConfig", "RequestMetrics", "RoutingDecision", "RunReport", "StepRecord", "SyntheticSpec",
    "TraceError", "TraceRecord", "UnsupportedConfigError", "chain_keys", "class_key", "combine64",
    "generate_synthetic", "generate_synthetic_packed", "load_trace", "percentile", "probe_capacity", "run", "save_trace",
    "scale_trace", "splitmix64", "stable_key", "export", "summarize", "load_trace_packed", "save_packed", "load_packed",
]
