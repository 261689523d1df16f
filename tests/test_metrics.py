"""metrics.summarize / export over the Collector columns vs the reference's exports
(tests/golden/metrics_exports.json: sha256 of every file the reference's
metrics.export wrote for the same run, tools/make_metrics_golden.py).

CPU: the report is assembled from the oracle's replay (same columns the device
writes). GPU: the report of a device replay through the public API."""
import hashlib
import json
import os

import numpy as np
import pytest

import golden_cases as G
from oracle.oracle import run_oracle
from paper_2603_15202_b200.metrics import export, summarize
from paper_2603_15202_b200.report import DetectorRow, RunReport

GOLD = json.load(open(os.path.join(G.GOLDEN, "metrics_exports.json")))


def report_from_oracle(trace, cfg) -> RunReport:
    o = run_oracle(trace, cfg, with_log=True)
    log = o.log
    routes = log[log[:, 0] == 0]
    steps = log[log[:, 0] == 1]
    idx = np.zeros(len(steps), np.int64)
    seen = {}
    for j, i in enumerate(steps[:, 1].tolist()):                 # per-instance step index
        idx[j] = seen.get(i, 0)
        seen[i] = idx[j] + 1
    step_log = np.stack([steps[:, 1], steps[:, 2], steps[:, 3], steps[:, 4], steps[:, 5], idx], axis=1)
    cols = {"chosen": o.chosen, "hit_tokens": o.hit_tokens, "first_sched_us": o.first_sched_us,
            "first_token_us": o.first_token_us, "finish_us": o.finish_us, "route_bs": routes[:, 5]}
    rep = RunReport(cfg.policy.kind, cfg.seed, cfg.n_instances, cfg.cache.block_size, trace=trace, columns=cols,
                    step_log=step_log, end_us=o.end_us, queued_at_last_arrival=o.queued_at_last_arrival)
    if cfg.detector is not None:
        rep.detector_enabled = True
        rep.detector_rows = [DetectorRow(*r) for r in o.detector_rows]
        rep.first_violation_us = o.first_violation_us if hasattr(o, "first_violation_us") else None
    return rep


def _check(rep, name, tmp_path):
    want = GOLD[name]
    got = {}
    for rw in (False, True):
        d = tmp_path / ("rw" if rw else "plain")
        for p in export(rep, d, request_weighted_hits=rw):
            got[f"{'rw/' if rw else ''}{os.path.basename(p)}"] = hashlib.sha256(open(p, "rb").read()).hexdigest()
    bad = sorted(k for k in want["files"] if got.get(k) != want["files"][k])
    assert not bad, f"{name}: files differ from the reference's export: {bad}"
    assert set(got) == set(want["files"])
    assert json.dumps(summarize(rep), indent=2, sort_keys=True) + "\n" == want["summary"]


@pytest.mark.parametrize("name", sorted(GOLD))
def test_export_from_oracle_columns(tmp_path, name):
    trace, cfg = G.build(name)
    _check(report_from_oracle(trace, cfg), name, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
def test_export_from_device_replay(tmp_path, name):
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.cluster import run
    _native.lib()
    trace, cfg = G.build(name)
    _check(run(trace, cfg), name, tmp_path)
