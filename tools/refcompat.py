"""Helpers to drive the *reference* routesim from this repo's traces/configs.

Used only by tools/make_golden.py and CPU-side cross-checks in this
container (the reference is not present on the GPU box).
"""
from __future__ import annotations

import os
import sys

REF_SRC = os.environ.get("ROUTESIM_SRC", "/root/reference/pkg/src")


def import_reference():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import routesim  # noqa: F401
    return routesim


def to_ref_config(cfg):
    rs = import_reference()
    from routesim.cluster import CacheConfig, ClusterConfig
    from routesim.detector import DetectorConfig
    from routesim.engine import CostModel
    from routesim.policies import PolicyConfig
    cm = cfg.cost_model
    return ClusterConfig(
        n_instances=cfg.n_instances,
        cost_model=CostModel(cm.prefill_base_ms, cm.prefill_per_token_ms, cm.decode_base_ms,
                             cm.decode_per_seq_ms, cm.decode_per_ctx_token_ms, cm.chunk_tokens,
                             cm.max_batch_requests),
        cache=CacheConfig(cfg.cache.block_size, cfg.cache.capacity_blocks),
        policy=PolicyConfig(**{k: getattr(cfg.policy, k) for k in cfg.policy.__dataclass_fields__}),
        staleness_ms=cfg.staleness_ms, seed=cfg.seed, parallel_instances=cfg.parallel_instances,
        detector=None if cfg.detector is None else DetectorConfig(
            **{k: getattr(cfg.detector, k) for k in cfg.detector.__dataclass_fields__}),
    )


def to_ref_records(trace):
    import_reference()
    from routesim.trace import TraceRecord
    out = []
    for r in trace.records():
        out.append(TraceRecord(r.request_id, r.arrival_s, r.prefix_blocks, r.input_tokens,
                               r.output_tokens, r.class_key))
    return out
