"""Generate golden fixtures by running the REFERENCE routesim in this container.

    python tools/make_golden.py            # writes tests/golden/*.npz

Each fixture stores the workload recipe (so tests can rebuild the identical
trace with ``paper_2603_15202_b200.workloads``), a fingerprint of the packed
trace, and the reference's outputs: per-request chosen instance, hit tokens,
first-sched / first-token / finish times, the step log, end_us,
queued_at_last_arrival and finished. Hash known-answer values come from the
reference's ``routesim.hashing``.

/root/reference is absent on the GPU box; the committed fixtures travel
instead.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from refcompat import import_reference, to_ref_config, to_ref_records  # noqa: E402

from paper_2603_15202_b200 import workloads as W  # noqa: E402
from paper_2603_15202_b200.config import (CacheConfig, ClusterConfig, CostModel,  # noqa: E402
                                          DetectorConfig, PolicyConfig)

OUT = os.path.join(ROOT, "tests", "golden")


def fingerprint(trace) -> str:
    h = hashlib.sha256()
    for a in (trace.request_id, trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.blk_off,
              trace.blocks):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# Recipes: name -> (builder expression, prefix length or None). The builder is
# evaluated against paper_2603_15202_b200.workloads / .config by tests/golden_cases.py.
CASES = {
    "cfg1_chatbot_full": ("W.config1_chatbot()", None),
    "cfg2_api_prefix4000": ("W.config2_api()", 4000),
    "cfg3_agent_prefix1200": ("W.config3_agent(1200)", None),
    "cfg3_agent_evict_n16": ("W.config3_agent(1500, n_instances=16, capacity=4096, rate_per_instance=1.0)", None),
    "cfg4_large_prefix300": ("W.config4_large(20000)", 300),
    "chat1024_prefix800": ("W.chat_cluster(1024, 3000)", 800),
    "adv_same_time_ties": ("W.adversarial('same_time_ties', 16, 0)", None),
    "adv_zero_bs": ("W.adversarial('zero_bs', 16, 0)", None),
    "adv_full_hits": ("W.adversarial('full_hits', 16, 0)", None),
    "adv_ragged": ("W.adversarial('ragged', 16, 0)", None),
    "adv_out1": ("W.adversarial('out1', 16, 0)", None),
    "adv_step_boundary": ("W.adversarial('step_boundary', 16, 0)", None),
    "adv_tight_capacity": ("W.adversarial('tight_capacity', 16, 0)", None),
    "adv_mixed_n16": ("W.adversarial('mixed', 16, 0)", None),
    # BASELINE configs[4] at bench scale (the bench line's adv64 workload): ties, bs 0, full hits,
    # out = 1, ragged inputs, repeated timestamps and tight-capacity evictions, interleaved
    "adv_stream_prefix6000": ("W.adversarial_stream()", 6000),
    "adv_mixed_n3": ("W.adversarial('mixed', 3, 1)", None),
    "adv_mixed_n33": ("W.adversarial('mixed', 33, 2)", None),
    "adv_mixed_n64": ("W.adversarial('mixed', 64, 3)", None),
    "evict_heavy_n4": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=4, cache=CacheConfig(16, 300), seed=5))", 1500),
    "policy_vllm": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, cache=CacheConfig(16, None), policy=PolicyConfig(kind='vllm'), seed=2))", 1000),
    "policy_least_bs": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='least_bs'), seed=3))", 1000),
    "policy_omh_total": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kv_indicator='one_minus_hit', balance_indicator='total_tokens'), seed=3))", 1000),
    "policy_omh_bs": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=12, policy=PolicyConfig(kv_indicator='one_minus_hit', tie_break_seed=9), seed=1))", 1000),
    "policy_linear": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='linear'), seed=4))", 1000),
    "policy_linear_cap": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=12, policy=PolicyConfig(kind='linear', kv_weight=0.7, bs_norm_cap=6), seed=5))", 1000),
    "policy_filter": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='filter'), seed=6))", 1000),
    "policy_filter_r2": ("(W.config2_api()[0], ClusterConfig(n_instances=16, policy=PolicyConfig(kind='filter', range_threshold=2, tie_break_seed=3), seed=7))", 1500),
    "policy_simulate": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='simulate'), seed=13))", 1000),
    "policy_simulate_mistuned": ("(W.config2_api()[0], ClusterConfig(n_instances=16, policy=PolicyConfig(kind='simulate', mis_tuned=True, tie_break_seed=5), seed=14))", 1500),
    "policy_simulate_factor": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=12, policy=PolicyConfig(kind='simulate', mis_tuned=True, mis_tuned_factor=0.37), staleness_ms=10.0, seed=15))", 1000),
    "policy_simulate_small_batch": ("(W.config2_api()[0], ClusterConfig(n_instances=4, cost_model=CostModel(1.0, 0.2, 4.0, 0.5, 0.01, 300, 3), cache=CacheConfig(16, 5000), policy=PolicyConfig(kind='simulate'), seed=16))", 800),
    "policy_simulate_agent_evict": ("(W.config3_agent(600, n_instances=16, capacity=4096, rate_per_instance=1.0)[0], ClusterConfig(n_instances=16, cache=CacheConfig(16, 4096), policy=PolicyConfig(kind='simulate'), seed=17))", None),
    "stale_5ms": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, staleness_ms=5.0, seed=8))", 1000),
    "stale_50ms_n16": ("(W.config2_api()[0], ClusterConfig(n_instances=16, staleness_ms=50.0, seed=9))", 1500),
    "stale_frac_vllm": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='vllm'), staleness_ms=12.3456, seed=10))", 1000),
    "stale_linear": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, policy=PolicyConfig(kind='linear'), staleness_ms=20.0, seed=11))", 1000),
    "stale_filter_evict": ("(W.config3_agent(1500, n_instances=16, capacity=4096, rate_per_instance=1.0)[0], ClusterConfig(n_instances=16, cache=CacheConfig(16, 4096), policy=PolicyConfig(kind='filter'), staleness_ms=100.0, seed=12))", None),
    "det_hot_n16": ("(lambda t, c: (t, dataclasses.replace(c, detector=DetectorConfig(window_s=5.0))))(*W.hotspot(16, 2000))", None),
    "det_hot_force_mean": ("(lambda t, c: (t, dataclasses.replace(c, detector=DetectorConfig(window_s=3.0, mitigation='force_least_bs', compare_mean_non_holder=True, consecutive_multiplier=1.0))))(*W.hotspot(12, 2000, 0.7, seed=4))", None),
    "det_hot_vllm_stale": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='vllm'), staleness_ms=20.0, detector=DetectorConfig(window_s=4.0, top_k_classes=2))))(*W.hotspot(8, 1500, 0.5, seed=5))", None),
    "det_chat_default": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=16, cache=CacheConfig(16, 40000), detector=DetectorConfig(), seed=0))", 1500),
    "det_api_k1": ("(W.config2_api()[0], ClusterConfig(n_instances=64, cache=CacheConfig(16, 40000), detector=DetectorConfig(window_s=2.0, top_k_classes=4, class_key_blocks=1), seed=0))", 3000),
    "det_simulate_n12": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='simulate'), detector=DetectorConfig(window_s=3.0, consecutive_multiplier=1.0))))(*W.hotspot(12, 1500, 0.7, seed=8))", None),
    "det_simulate_force": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='simulate', mis_tuned=True), detector=DetectorConfig(window_s=2.0, mitigation='force_least_bs', consecutive_multiplier=1.0))))(*W.hotspot(10, 1500, 0.75, seed=9))", None),
    "det_filter_n12": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='filter', range_threshold=2), detector=DetectorConfig(window_s=3.0, consecutive_multiplier=1.0))))(*W.hotspot(12, 1500, 0.7, 120.0, seed=10))", None),
    "det_filter_force": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='filter'), detector=DetectorConfig(window_s=2.0, mitigation='force_least_bs', consecutive_multiplier=0.5, compare_mean_non_holder=True))))(*W.hotspot(16, 2000, 0.8, 200.0, seed=11))", None),
    "det_linear_uncapped": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='linear', kv_weight=0.3), detector=DetectorConfig(window_s=3.0, consecutive_multiplier=1.0))))(*W.hotspot(12, 1500, 0.7, 150.0, seed=12))", None),
    "det_linear_stale": ("(lambda t, c: (t, dataclasses.replace(c, policy=PolicyConfig(kind='linear'), staleness_ms=15.0, detector=DetectorConfig(window_s=2.0, consecutive_multiplier=0.5, compare_mean_non_holder=True))))(*W.hotspot(16, 2000, 0.8, 250.0, seed=13))", None),
    "det_evict_n8": ("(lambda t, c: (t, dataclasses.replace(c, cache=CacheConfig(16, 600), detector=DetectorConfig(window_s=2.0, consecutive_multiplier=0.5))))(*W.hotspot(8, 2000, 0.8, 90.0, seed=6))", None),
    "cost_fma_sensitive": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, cost_model=CostModel(3.3, 0.0371, 17.1, 0.77, 0.0013, 512, 16), cache=CacheConfig(16, 2000), seed=4))", 1000),
    "cost_small_batch": ("(W.config2_api()[0], ClusterConfig(n_instances=6, cost_model=CostModel(1.0, 0.2, 4.0, 0.5, 0.01, 300, 3), cache=CacheConfig(16, 5000), seed=7))", 1500),
    "block_size_4": ("W.generate_synthetic_packed(W.SyntheticSpec(60.0, 20.0, (W.ClassSpec(0.5, 6, (1, 5), (1, 30)), W.ClassSpec(0.5, 2, (0, 3), (1, 9))), seed=11, block_size=4)), ClusterConfig(n_instances=5, cache=CacheConfig(4, 500), seed=11)", None),
}


def build_case(expr: str, prefix):
    env = {"dataclasses": dataclasses, "W": W, "ClusterConfig": ClusterConfig, "CacheConfig": CacheConfig, "CostModel": CostModel,
           "PolicyConfig": PolicyConfig, "DetectorConfig": DetectorConfig}
    trace, cfg = eval(expr, env)
    if prefix is not None:
        trace = trace.slice(min(prefix, len(trace)))
    return trace, cfg


def run_reference(trace, cfg):
    rs = import_reference()
    t0 = time.perf_counter()
    rep = rs.run(to_ref_records(trace), to_ref_config(cfg))
    dt = time.perf_counter() - t0

    def col(name):
        return np.asarray([-1 if getattr(r, name) is None else getattr(r, name) for r in rep.requests],
                          dtype=np.int64)

    steps = np.asarray([(s.instance, s.start_us, s.end_us, s.prefill_us) for s in rep.steps],
                       dtype=np.int64).reshape(-1, 4)
    det = {}
    if rep.detector_enabled:
        rows = rep.detector_rows
        det = dict(
            det_window_start_s=np.asarray([r.window_start_s for r in rows], np.float64),
            det_class_key=np.asarray([r.class_key for r in rows], np.uint64),
            det_fraction=np.asarray([r.fraction for r in rows], np.float64),
            det_ints=np.asarray([(r.n_holders, r.n_others, int(r.suspect), r.phase) for r in rows],
                                np.int64).reshape(-1, 4),
            det_first_violation_us=np.asarray([-1 if rep.first_violation_us is None else rep.first_violation_us],
                                              np.int64))
    return dict(
        **det,
        chosen=np.asarray([r.chosen_instance for r in rep.requests], dtype=np.int32),
        hit_tokens=col("hit_tokens"), first_sched_us=col("first_sched_us"),
        first_token_us=col("first_token_us"), finish_us=col("finish_us"), steps=steps,
        summary=np.asarray([rep.end_us, rep.queued_at_last_arrival, rep.finished, rep.routed],
                           dtype=np.int64),
    ), dt


def kats():
    rs = import_reference()
    from routesim import hashing as h
    from routesim.detector import class_key
    vals = [0, 1, 2, 0x9E3779B97F4A7C15, (1 << 64) - 1, 12345678901234567, 1 << 63]
    return {
        "splitmix64": [[v, h.splitmix64(v)] for v in vals],
        "combine64": [[a, b, h.combine64(a, b)] for a in vals[:4] for b in vals[:4]],
        "stable_key": [[list(t), h.stable_key(*t)] for t in
                       [(0, 0), (1, 0), (0x0F0C0DE, 7, 0), (0x0F0C0DE, 0, 0), (0, 1), (5, 9), (2**64 - 1,)]],
        "chain_keys": [[list(b), h.chain_keys(b)] for b in
                       [[1, 2, 3], [0], list(range(40)), [2**64 - 1, 0, 2**63]]],
        "class_key": [[list(b), class_key(b)] for b in [[1, 2, 3], [7], [9, 9]]],
        "_source": "routesim.hashing / routesim.detector.class_key run in this container",
    }


def main(only=None):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "hash_kats.json"), "w") as fh:
        json.dump(kats(), fh, indent=1)
    index = {}
    for name, (expr, prefix) in CASES.items():
        if only and name not in only:
            continue
        trace, cfg = build_case(expr, prefix)
        out, dt = run_reference(trace, cfg)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        index[name] = {"expr": expr, "prefix": prefix, "n_requests": len(trace),
                       "fingerprint": fingerprint(trace), "reference_seconds": round(dt, 3)}
        print(f"{name:28s} R={len(trace):6d}  ref {dt:7.2f}s", flush=True)
    path = os.path.join(OUT, "index.json")
    old = json.load(open(path)) if (only and os.path.exists(path)) else {}
    old.update(index)
    with open(path, "w") as fh:
        json.dump(old, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
