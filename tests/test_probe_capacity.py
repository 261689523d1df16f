"""probe_capacity (reference cluster.py:295-330) against values the reference itself
produced (tests/golden/probe_capacity.json, tools/make_probe_golden.py).

CPU: the same search with every probe replayed by the oracle (checks scale_packed and
the search). GPU: the drop-in, every probe a device replay through librsim."""
import json
import os

import numpy as np
import pytest

import golden_cases as G
from oracle.oracle import run_oracle

GOLDEN = json.load(open(os.path.join(G.GOLDEN, "probe_capacity.json")))


def _build(meta):
    import dataclasses
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, CostModel, PolicyConfig
    env = {"dataclasses": dataclasses, "W": W, "ClusterConfig": ClusterConfig, "CacheConfig": CacheConfig,
           "CostModel": CostModel, "PolicyConfig": PolicyConfig}
    trace, cfg = eval(meta["expr"], env)
    return trace.slice(min(meta["prefix"], len(trace))), cfg


def test_scale_packed_matches_scale_trace():
    from paper_2603_15202_b200.trace import scale_packed, scale_trace
    trace, _ = _build(GOLDEN["chat_n4_mb4"])
    for rate in (0.5, 9.28125, 333.0):
        a = scale_packed(trace, rate)
        b = scale_trace(trace.records(), rate)
        assert np.array_equal(a.arrival_s, np.array([r.arrival_s for r in b]))
        assert np.array_equal(a.arrival_us, np.rint(np.array([r.arrival_s for r in b]) * 1e6).astype(np.int64))


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_probe_search_with_oracle(name, monkeypatch):
    from paper_2603_15202_b200 import cluster
    meta = GOLDEN[name]
    trace, cfg = _build(meta)
    monkeypatch.setattr(cluster, "run", lambda tr, c, **kw: run_oracle(tr, c))
    assert cluster.probe_capacity(trace, cfg, **meta["kwargs"]) == meta["capacity_rps"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_probe_capacity_on_device(name):
    from paper_2603_15202_b200 import _native, probe_capacity
    _native.lib()
    meta = GOLDEN[name]
    trace, cfg = _build(meta)
    assert probe_capacity(trace, cfg, **meta["kwargs"]) == meta["capacity_rps"]
