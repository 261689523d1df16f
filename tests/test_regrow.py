"""Capacity regrow paths: a per-instance queue ring, KV$ table or LRU
touch-run ring sized too small is detected on the device (RSIM_E_QUEUE_OVERFLOW /
RSIM_E_TABLE_FULL), and the public API rebuilds a larger handle and replays -- the decisions are
the reference's either way (golden fixtures recorded from reference run(), cluster.py:290-292)."""
import dataclasses

import pytest

import golden_cases as G

pytestmark = pytest.mark.gpu


def _handle_error(name, **fields):
    """Replay fixture `name` on a raw handle with some native config fields forced; return the
    CapacityError it raises."""
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.cluster import native_config, sizing_for
    trace, cfg = G.build(name)
    c = native_config(cfg, sizing_for(trace, cfg))
    for k, v in fields.items():
        setattr(c, k, v)
    h = _native.Handle(c)
    try:
        h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
        with pytest.raises(_native.CapacityError) as ei:
            h.rerun()
        return ei.value
    finally:
        h.close()


def test_queue_ring_overflow_is_reported():
    from paper_2603_15202_b200 import _native
    e = _handle_error("cost_small_batch", queue_capacity=16)
    assert e.status == _native.E_QUEUE_OVERFLOW and "queue ring" in str(e)


def test_table_overflow_is_reported():
    from paper_2603_15202_b200 import _native
    e = _handle_error("cfg2_api_prefix4000", expected_keys=64)
    assert e.status == _native.E_TABLE_FULL and "KV$ table" in str(e)


def test_touch_run_ring_overflow_is_reported():
    from paper_2603_15202_b200 import _native
    e = _handle_error("cfg1_chatbot_full", runs_capacity=64)
    assert e.status == _native.E_TABLE_FULL and "touch-run ring" in str(e)


@pytest.mark.parametrize("name,sizing", [
    ("cost_small_batch", dict(queue_capacity=16)),
    ("cfg2_api_prefix4000", dict(expected_keys=64)),
    ("evict_heavy_n4", dict(queue_capacity=16, expected_keys=16)),      # runs ring derives from the queue
    ("cfg3_agent_evict_n16", dict(queue_capacity=16, expected_keys=256)),
])
def test_regrown_replay_matches_reference(name, sizing, monkeypatch):
    """run() starting from rings/tables far too small: every overflow regrows and the final
    replay is bit-identical to the reference's."""
    from paper_2603_15202_b200 import cluster
    from test_device_parity import _assert_report
    real = cluster.sizing_for
    grown = []
    real_rebuild = cluster.ClusterSim._rebuild

    def rebuild(self, *a, **k):
        grown.append(self._sizing)
        return real_rebuild(self, *a, **k)

    monkeypatch.setattr(cluster, "sizing_for", lambda t, c: dataclasses.replace(real(t, c), **sizing))
    monkeypatch.setattr(cluster.ClusterSim, "_rebuild", rebuild)
    cluster._LEARNED.clear()
    try:
        trace, cfg = G.build(name)
        rep = cluster.run(trace, cfg)
    finally:
        cluster._LEARNED.clear()
        cluster.release_pool()
    assert grown, "the undersized replay never overflowed"
    _assert_report(rep, G.expected(name), name)

