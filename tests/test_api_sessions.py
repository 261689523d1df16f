"""Stateful drop-in API sessions against the reference (tests/golden/api_sessions.json, made by
tools/make_api_golden.py from the reference's ClusterSim): route() / enqueue() / cache.insert()
followed by run_trace(), run_trace() twice on one sim (state and Collector persist,
cluster.py:98-201), duplicate request ids (DuplicateRequestError after the tie-break,
engine.py:266-267), and the instance queues (engine.py:212-213)."""
import json
import os
import sys

import pytest

import golden_cases as G

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def _ours():
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import DuplicateRequestError
    return ClusterSim, (lambda tr: tr.records()), DuplicateRequestError


@pytest.mark.parametrize("name", ["route_then_run", "run_twice", "duplicates", "duplicates_then_run", "enqueue_dup",
                                  "small_batch_queues"])
def test_session_matches_reference(name):
    import make_api_golden as M
    from paper_2603_15202_b200 import workloads as W
    want = json.load(open(os.path.join(G.GOLDEN, "api_sessions.json")))[name]
    cfg, steps = M.SESSIONS[name]
    trace = W.config1_chatbot()[0].slice(600)
    got = M.run_session(cfg, steps, trace, _ours())
    got = json.loads(json.dumps(got))
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"step {i} ({steps[i]}): {str(g)[:300]} != {str(w)[:300]}"


def test_session_survives_regrow():
    """A queue ring too small for the API calls: the sim regrows the handle by replaying its
    logged calls, and the session still matches the reference."""
    import make_api_golden as M
    from paper_2603_15202_b200 import cluster, workloads as W
    want = json.load(open(os.path.join(G.GOLDEN, "api_sessions.json")))["small_batch_queues"]
    cfg, steps = M.SESSIONS["small_batch_queues"]
    trace = W.config1_chatbot()[0].slice(600)
    real = cluster.sizing_for
    try:
        cluster.sizing_for = lambda t, c: cluster.Sizing(16, 64) if t is None else real(t, c)
        cluster._LEARNED.clear()
        got = json.loads(json.dumps(M.run_session(cfg, steps, trace, _ours())))
    finally:
        cluster.sizing_for = real
        cluster._LEARNED.clear()
    assert got == want


@pytest.mark.parametrize("name", ["det_exclude", "det_force_least_bs", "det_enqueue_mix", "det_many_instances",
                                  "det_dup_new_class"])
def test_detector_route_session_matches_reference(name):
    """route() with the prefix-hotspot detector (cluster.py:133-139: verdict before choose, observe
    after the enqueue) on the device: holders made by cache.insert(), the hot trace routed call by
    call -- suspects, phase-2 streaks, alarms and both mitigations show in the decisions (each
    session routes >= 55 requests differently from the same session without the detector)."""
    import make_api_golden as M
    from paper_2603_15202_b200 import workloads as W
    want = json.load(open(os.path.join(G.GOLDEN, "api_sessions.json")))[name]
    cfg, (holders, n_route, extra) = M.DET_SESSIONS[name]
    hot = W.hotspot(8, 600, 0.6, 20.0, seed=4)[0]
    steps = M._hot_steps(hot, holders, n_route, extra)
    got = json.loads(json.dumps(M.run_session(cfg, steps, hot, _ours())))
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"step {i} ({steps[i]}): {str(g)[:300]} != {str(w)[:300]}"


def test_detector_route_session_survives_regrow():
    """The detector session on rings too small: every regrow replays the logged route() calls
    (with their detector classes) onto a fresh handle, and the decisions still match."""
    import make_api_golden as M
    from paper_2603_15202_b200 import cluster, workloads as W
    want = json.load(open(os.path.join(G.GOLDEN, "api_sessions.json")))["det_exclude"]
    cfg, (holders, n_route, extra) = M.DET_SESSIONS["det_exclude"]
    hot = W.hotspot(8, 600, 0.6, 20.0, seed=4)[0]
    steps = M._hot_steps(hot, holders, n_route, extra)
    real = cluster.sizing_for
    try:
        cluster.sizing_for = lambda t, c: cluster.Sizing(16, 64) if t is None else real(t, c)
        cluster._LEARNED.clear()
        got = json.loads(json.dumps(M.run_session(cfg, steps, hot, _ours())))
    finally:
        cluster.sizing_for = real
        cluster._LEARNED.clear()
    assert got == want


def test_run_trace_refused_while_an_id_is_live_on_two_instances():
    """The reference's Collector files every event under the newest RequestMetrics of an id
    (metrics.py:116-139): once one id is live on two instances, the per-copy device columns would
    report differently, so run_trace refuses (UnsupportedConfigError) instead of diverging."""
    import make_api_golden as M
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.config import UnsupportedConfigError
    ClusterSim, conv, Dup = _ours()
    cfg, steps = M.SESSIONS["duplicates"]
    trace = W.config1_chatbot()[0].slice(600)
    recs = conv(trace)
    sim = ClusterSim(cfg)
    sim.route(recs[0], int(trace.arrival_us[0]))
    placed = 1
    for j in range(1, 40):                   # until the id lands on a second instance
        try:
            sim.route(recs[0], 70_000 + j)
            placed += 1
            break
        except Dup:
            pass
    assert placed == 2
    with pytest.raises(UnsupportedConfigError):
        sim.run_trace(recs[300:320])


@pytest.mark.parametrize("name", ["fuzz_mult_n5", "fuzz_vllm_n12", "fuzz_linear_n3", "fuzz_filter_n7", "fuzz_mult_n300"])
def test_fuzz_session_matches_reference(name):
    """Seeded random API sessions (route, repeated ids, enqueue, cache.insert, queue views) on
    the one-launch route path (plain policies, <= 256 instances) and the three-launch path
    (filter, 300 instances), against the reference's ClusterSim."""
    import make_api_golden as M
    from paper_2603_15202_b200 import workloads as W
    want = json.load(open(os.path.join(G.GOLDEN, "api_sessions.json")))[name]
    cfg, seed = M.FUZZ_SESSIONS[name]
    steps = M._fuzz_steps(seed, cfg.n_instances)
    trace = W.config1_chatbot()[0].slice(600)
    got = json.loads(json.dumps(M.run_session(cfg, steps, trace, _ours())))
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        assert g == w, f"step {i} ({steps[i]}): {str(g)[:300]} != {str(w)[:300]}"
