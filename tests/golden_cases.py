"""Golden fixtures produced by running the reference (tools/make_golden.py).

Each case is rebuilt from its recipe with this repo's workload builders and
checked against the recorded trace fingerprint before use, so a fixture can
never silently be compared against a different trace.
"""
import hashlib
import json
import os

import numpy as np

from paper_2603_15202_b200 import workloads as W
import dataclasses

from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, CostModel, DetectorConfig, PolicyConfig

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index():
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)


def fingerprint(trace) -> str:
    h = hashlib.sha256()
    for a in (trace.request_id, trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.blk_off, trace.blocks):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def build(name: str):
    meta = index()[name]
    env = {"dataclasses": dataclasses, "W": W, "ClusterConfig": ClusterConfig, "CacheConfig": CacheConfig,
           "CostModel": CostModel, "PolicyConfig": PolicyConfig, "DetectorConfig": DetectorConfig}
    trace, cfg = eval(meta["expr"], env)
    if meta["prefix"] is not None:
        trace = trace.slice(min(meta["prefix"], len(trace)))
    assert fingerprint(trace) == meta["fingerprint"], f"{name}: trace drifted from the golden recipe"
    return trace, cfg


def expected(name: str) -> dict:
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def names(max_requests: int | None = None):
    idx = index()
    return sorted(n for n, m in idx.items() if max_requests is None or m["n_requests"] <= max_requests)


def kats() -> dict:
    with open(os.path.join(GOLDEN, "hash_kats.json")) as fh:
        return json.load(fh)


def detector_rows(want: dict):
    """The reference's DetectorRow list of a detector fixture as tuples
    (window_start_s, class_key, fraction, n_holders, n_others, suspect, phase)."""
    ints = want["det_ints"]
    return [(float(want["det_window_start_s"][i]), int(want["det_class_key"][i]), float(want["det_fraction"][i]),
             int(ints[i, 0]), int(ints[i, 1]), bool(ints[i, 2]), int(ints[i, 3])) for i in range(len(ints))]


def first_violation(want: dict):
    v = int(want["det_first_violation_us"][0])
    return None if v < 0 else v


def random_detector_case(seed: int, trial: int):
    """Trial ``trial`` of the random detector parity sweep (test_device_parity.py): a
    hotspot trace and a random detector / policy / cache / staleness configuration."""
    rng = np.random.default_rng(500 + seed)
    for _ in range(trial + 1):
        N = int(rng.choice([3, 8, 16, 40, 100]))
        trace, cfg = W.hotspot(N, int(rng.integers(300, 1500)), float(rng.uniform(0.3, 0.9)),
                               float(rng.uniform(20, 200)), int(rng.integers(1, 12)), seed=int(rng.integers(0, 99)))
        kind = str(rng.choice(["multiplicative", "multiplicative", "vllm", "least_bs", "linear"]))
        pol = PolicyConfig(kind=kind, kv_indicator=str(rng.choice(["p_tokens", "one_minus_hit"])),
                           balance_indicator=str(rng.choice(["bs", "total_tokens"])),
                           bs_norm_cap=int(rng.integers(1, 9)) if kind == "linear" else None,
                           tie_break_seed=int(rng.integers(0, 9)))
        det = DetectorConfig(window_s=float(rng.choice([0.5, 1.0, 2.5, 7.0, 60.0])),
                             top_k_classes=int(rng.integers(1, 6)), class_key_blocks=int(rng.integers(1, 4)),
                             consecutive_multiplier=float(rng.choice([0.0, 0.5, 1.0, 2.0])),
                             mitigation=str(rng.choice(["exclude_holders", "force_least_bs"])),
                             compare_mean_non_holder=bool(rng.integers(0, 2)))
        cap = [None, int(rng.integers(200, 2000))][int(rng.integers(0, 2))]
        cfg = dataclasses.replace(cfg, policy=pol, detector=det, cache=CacheConfig(16, cap),
                                  staleness_ms=float(rng.choice([0.0, 0.0, 7.5])))
    return trace, cfg
