"""Device parity: librsim on the B200 against the reference's golden outputs
and the oracle. Bit-exact (integer/index work): decisions, hit tokens, per-
request first-sched / first-token / finish times, the step log and the run
summary."""
import numpy as np
import pytest

import golden_cases as G
from oracle.oracle import OracleCache, run_oracle
from oracle.oracle import chain_keys as oracle_chain_keys

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_2603_15202_b200 import _native
    _native.lib()
    return _native


def _assert_report(rep, want, name):
    c = rep.columns
    for key in ("chosen", "hit_tokens", "first_sched_us", "first_token_us", "finish_us"):
        got = c[key]
        if not np.array_equal(got, want[key]):
            i = int(np.nonzero(got != want[key])[0][0])
            raise AssertionError(f"{name}: {key} differs first at request {i}: {got[i]} != {want[key][i]}")
    steps = np.asarray([(s.instance, s.start_us, s.end_us, s.prefill_us) for s in rep.steps],
                       np.int64).reshape(-1, 4)
    assert np.array_equal(steps, want["steps"]), f"{name}: step log differs"
    s = want["summary"]
    assert (rep.end_us, rep.queued_at_last_arrival, rep.finished, rep.routed) == tuple(int(x) for x in s[:4])
    if "det_ints" in want:                          # detector rows + first violation (detector.py:340-377)
        rows = [(r.window_start_s, r.class_key, r.fraction, r.n_holders, r.n_others, r.suspect, r.phase)
                for r in rep.detector_rows]
        assert rows == G.detector_rows(want), f"{name}: detector rows differ"
        assert rep.first_violation_us == G.first_violation(want), f"{name}: first violation differs"


@pytest.mark.parametrize("name", G.names())
def test_replay_matches_reference_golden(native, name):
    from paper_2603_15202_b200.cluster import run
    trace, cfg = G.build(name)
    rep = run(trace, cfg)
    _assert_report(rep, G.expected(name), name)


@pytest.mark.parametrize("shape", [(1, 2), (1, 4), (2, 8), (4, 2), (16, 1)])
def test_cluster_shapes_agree(native, shape):
    """The same decisions for every CTA-cluster / warp split of the instances."""
    from paper_2603_15202_b200.cluster import run
    trace, cfg = G.build("adv_mixed_n33")
    rep = run(trace, cfg, ctas=shape[0], warps_per_cta=shape[1])
    _assert_report(rep, G.expected("adv_mixed_n33"), f"shape{shape}")


def test_chain_keys_kats(native):
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import ClusterConfig
    sim = ClusterSim(ClusterConfig(n_instances=1))
    h = sim._device()
    for blocks, want in G.kats()["chain_keys"]:
        got = h.chain_keys(np.asarray(blocks, dtype=np.uint64))
        assert [int(x) for x in got] == want
    rng = np.random.default_rng(5)
    b = rng.integers(0, 2**63, size=5000, dtype=np.uint64)
    assert np.array_equal(h.chain_keys(b), oracle_chain_keys(b))
    sim.close()


@pytest.mark.parametrize("n,ctas", [(600, 0), (1024, 16)])
def test_detector_large_cluster_matches_oracle(native, n, ctas):
    """The detector across a whole multi-CTA cluster (> 256 instances) vs the oracle."""
    import dataclasses
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import run
    from paper_2603_15202_b200.config import DetectorConfig
    trace, cfg = W.hotspot(n, 3000, 0.6, 2.5 * n, seed=21)
    cfg = dataclasses.replace(cfg, detector=DetectorConfig(window_s=1.0, top_k_classes=4, consecutive_multiplier=1.0))
    ref = run_oracle(trace, cfg)
    rep = run(trace, cfg, ctas=ctas) if ctas else run(trace, cfg)
    assert np.array_equal(rep.chosen, ref.chosen)
    assert np.array_equal(rep.hit_tokens, ref.hit_tokens)
    rows = [(r.window_start_s, r.class_key, r.fraction, r.n_holders, r.n_others, r.suspect, r.phase)
            for r in rep.detector_rows]
    assert len(rows) > 0 and rows == ref.detector_rows


@pytest.mark.parametrize("seed", range(3))
def test_random_simulate_configs_match_oracle(native, seed):
    """The simulate policy (TTFT replay per candidate, policies.py:142-157) on random clusters,
    cost models (tight chunk / max_batch), capacities and mis-tuned factors vs the oracle
    (the oracle's simulate is pinned to the reference by the policy_simulate_* fixtures)."""
    from paper_2603_15202_b200.cluster import run
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, CostModel, PolicyConfig
    from paper_2603_15202_b200.trace import ClassSpec, SyntheticSpec, generate_synthetic_packed
    rng = np.random.default_rng(700 + seed)
    for trial in range(5):
        n_cls = int(rng.integers(1, 5))
        w = rng.random(n_cls) + 0.1
        w = w / w.sum()
        classes = tuple(ClassSpec(float(x), int(rng.integers(0, 12)),
                                  (int(a := rng.integers(1, 4)), int(a + rng.integers(0, 6))),
                                  (1, int(rng.integers(1, 120)))) for x in w)
        bs = int(rng.choice([4, 16]))
        spec = SyntheticSpec(float(rng.uniform(5, 30)), float(rng.uniform(5, 90)), classes,
                             seed=int(rng.integers(0, 1000)), block_size=bs)
        trace = generate_synthetic_packed(spec)
        if len(trace) == 0:
            continue
        N = int(rng.choice([1, 2, 3, 7, 16, 33, 70]))
        cap = [None, int(rng.integers(20, 400)), 40000][int(rng.integers(0, 3))]
        cm = CostModel(float(rng.uniform(0, 8)), float(rng.choice([0.1, 0.0371, 0.05])),
                       float(rng.uniform(0, 30)), float(rng.uniform(0, 2)), float(rng.choice([0.0, 0.001, 0.0013])),
                       int(rng.choice([40, 64, 512, 2048])), int(rng.choice([2, 8, 40, 256])))
        pol = PolicyConfig(kind="simulate", mis_tuned=bool(rng.integers(0, 2)),
                           mis_tuned_factor=float(rng.choice([4.0, 0.3, 1.7])),
                           tie_break_seed=int(rng.integers(0, 50)))
        cfg = ClusterConfig(n_instances=N, cost_model=cm, cache=CacheConfig(bs, cap), policy=pol,
                            staleness_ms=float(rng.choice([0.0, 3.0])), seed=int(rng.integers(0, 99)))
        ref = run_oracle(trace, cfg)
        rep = run(trace, cfg)
        tag = f"seed{seed}/trial{trial} N={N} cap={cap} chunk={cm.chunk_tokens} mb={cm.max_batch_requests}"
        assert np.array_equal(rep.chosen, ref.chosen), tag
        assert np.array_equal(rep.hit_tokens, ref.hit_tokens), tag
        assert np.array_equal(rep.columns["first_token_us"], ref.first_token_us), tag
        assert np.array_equal(rep.columns["finish_us"], ref.finish_us), tag


@pytest.mark.parametrize("seed", range(4))
def test_random_configs_match_oracle(native, seed):
    """Random cluster sizes, cost models, capacities and policies vs the oracle."""
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import run
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, CostModel, PolicyConfig
    from paper_2603_15202_b200.trace import ClassSpec, SyntheticSpec, generate_synthetic_packed
    rng = np.random.default_rng(100 + seed)
    for trial in range(6):
        n_cls = int(rng.integers(1, 6))
        w = rng.random(n_cls) + 0.1
        w = w / w.sum()
        classes = tuple(ClassSpec(float(x), int(rng.integers(0, 12)),
                                  (int(a := rng.integers(1, 4)), int(a + rng.integers(0, 6))),
                                  (1, int(rng.integers(1, 80)))) for x in w)
        bs = int(rng.choice([4, 16, 32]))
        spec = SyntheticSpec(float(rng.uniform(5, 40)), float(rng.uniform(5, 80)), classes,
                             seed=int(rng.integers(0, 1000)), block_size=bs)
        trace = generate_synthetic_packed(spec)
        if len(trace) == 0:
            continue
        N = int(rng.choice([1, 2, 3, 7, 16, 33, 70]))
        cap = [None, int(rng.integers(20, 400)), 40000][int(rng.integers(0, 3))]
        cm = CostModel(float(rng.uniform(0, 8)), float(rng.choice([0.1, 0.0371, 0.05])),
                       float(rng.uniform(0, 30)), float(rng.uniform(0, 2)), float(rng.choice([0.0, 0.001, 0.0013])),
                       int(rng.choice([64, 512, 2048])), int(rng.choice([2, 8, 256])))
        kind = str(rng.choice(["multiplicative", "multiplicative", "vllm", "least_bs", "linear", "filter"]))
        pol = PolicyConfig(kind=kind, kv_indicator=str(rng.choice(["p_tokens", "one_minus_hit"])),
                           balance_indicator=str(rng.choice(["bs", "total_tokens"])),
                           tie_break_seed=int(rng.integers(0, 50)), q_weight=float(rng.choice([1.0, 0.5])),
                           kv_weight=float(rng.choice([0.0, 0.4, 0.75, 1.0])),
                           bs_norm_cap=[None, 1, 3, 8, 64][int(rng.integers(0, 5))],
                           range_threshold=int(rng.choice([1, 2, 4, 9])))
        stal = float(rng.choice([0.0, 0.0, 0.5, 3.7, 25.0, 200.0]))
        cfg = ClusterConfig(n_instances=N, cost_model=cm, cache=CacheConfig(bs, cap), policy=pol,
                            staleness_ms=stal, seed=int(rng.integers(0, 99)))
        ref = run_oracle(trace, cfg)
        rep = run(trace, cfg)
        tag = f"seed{seed}/trial{trial} N={N} cap={cap} {kind} staleness={stal}"
        assert np.array_equal(rep.chosen, ref.chosen), tag
        assert np.array_equal(rep.hit_tokens, ref.hit_tokens), tag
        assert np.array_equal(rep.columns["first_token_us"], ref.first_token_us), tag
        assert np.array_equal(rep.columns["finish_us"], ref.finish_us), tag
        assert rep.end_us == ref.end_us and rep.queued_at_last_arrival == ref.queued_at_last_arrival, tag


@pytest.mark.parametrize("seed", range(3))
def test_random_detector_configs_match_oracle(native, seed):
    """Random hotspot traces and detector settings (window, top-k, class key blocks,
    mitigation, mean comparison, multiplier) under every detector-compatible score,
    with staleness and eviction, vs the oracle: decisions, rows, first violation."""
    from paper_2603_15202_b200.cluster import run
    for trial in range(4):
        trace, cfg = G.random_detector_case(seed, trial)
        ref = run_oracle(trace, cfg)
        rep = run(trace, cfg)
        tag = f"seed{seed}/trial{trial} {cfg}"
        assert np.array_equal(rep.chosen, ref.chosen), tag
        assert np.array_equal(rep.columns["finish_us"], ref.finish_us), tag
        rows = [(r.window_start_s, r.class_key, r.fraction, r.n_holders, r.n_others, r.suspect, r.phase)
                for r in rep.detector_rows]
        assert rows == ref.detector_rows, tag
        assert rep.first_violation_us == ref.first_violation_us, tag


@pytest.mark.parametrize("name", ["stale_50ms_n16", "stale_filter_evict"])
def test_stale_history_ring_small(native, name, monkeypatch):
    """A view-history ring far below the staleness window: entries no later
    snapshot can see are dropped on device, and a ring that still overflows is
    reported (RSIM_E_HISTORY_OVERFLOW) and regrown -- same decisions either way."""
    import dataclasses

    from paper_2603_15202_b200 import cluster
    real = cluster.sizing_for
    monkeypatch.setattr(cluster, "sizing_for", lambda t, c: dataclasses.replace(real(t, c), history_capacity=16))
    trace, cfg = G.build(name)
    rep = cluster.run(trace, cfg)
    _assert_report(rep, G.expected(name), name)


@pytest.mark.parametrize("cap", [None, 8, 32, 128])
def test_cache_random_ops_match_oracle(native, cap):
    """Random insert / match sequences on one device instance vs the oracle
    PrefixCache (reference test_kvcache.py:141-174 style)."""
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig
    sim = ClusterSim(ClusterConfig(n_instances=2, cache=CacheConfig(16, cap)))
    h = sim._device()
    ref = OracleCache(cap)
    rng = np.random.default_rng(7 if cap is None else cap)
    roots = [int(x) for x in rng.integers(1, 50, size=6)]
    for op in range(400):
        n = int(rng.integers(1, 10))
        blocks = [roots[int(rng.integers(0, len(roots)))]] + [int(x) for x in rng.integers(1, 6, size=n - 1)]
        keys = oracle_chain_keys(blocks)
        now = int(rng.integers(0, 50)) + op // 4
        if rng.random() < 0.6:
            assert h.cache_insert_keys(1, keys, now) == ref.insert_keys(keys, now), op
        else:
            assert h.cache_match_keys(1, keys) == ref.match_keys(keys), op
        if op % 50 == 0:
            assert int(h.instances()[1, 11]) == ref.occupancy
    sim.close()


def test_route_multiplicative_prefers_full_hit(native):
    """reference test_cluster.py:32-40"""
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, PolicyConfig
    from paper_2603_15202_b200.trace import TraceRecord
    sim = ClusterSim(ClusterConfig(n_instances=2, cache=CacheConfig(capacity_blocks=None),
                                   policy=PolicyConfig(kind="multiplicative")))
    blocks = tuple(range(1, 33))
    sim.instances[0].cache.insert(blocks, 0)
    d = sim.route(TraceRecord(0, 0.0, blocks, 500, 4, 0), 0)
    assert d.chosen == 0
    assert d.scores[0] == 1.0 and d.scores[1] == 500.0
    sim.close()


def test_route_tie_break_depends_only_on_seed(native):
    """reference test_cluster.py:43-54"""
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, PolicyConfig
    from paper_2603_15202_b200.trace import TraceRecord
    rec = TraceRecord(0, 0.0, (1, 2), 32, 4, 0)

    def pick(seed):
        sim = ClusterSim(ClusterConfig(n_instances=2, cache=CacheConfig(capacity_blocks=None),
                                       policy=PolicyConfig(kind="vllm"), seed=seed))
        c = sim.route(rec, 0).chosen
        sim.close()
        return c
    first = {s: pick(s) for s in range(4)}
    assert first == {s: pick(s) for s in range(4)}
    assert set(first.values()) == {0, 1}


def test_enqueue_then_route_vllm(native):
    """reference test_cluster.py:57-70"""
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, PolicyConfig
    from paper_2603_15202_b200.trace import TraceRecord
    sim = ClusterSim(ClusterConfig(n_instances=3, cache=CacheConfig(capacity_blocks=None),
                                   policy=PolicyConfig(kind="vllm")))
    rid = 0
    for inst, n in enumerate((4, 2, 7)):
        for _ in range(n):
            sim.instances[inst].enqueue(TraceRecord(rid, 0.0, (rid + 1,), 16, 4, 0), 0)
            rid += 1
    assert sim.route(TraceRecord(99, 0.0, (1000,), 16, 4, 0), 0).chosen == 1
    sim.close()


def test_probe_batch_matches_oracle_cache(native):
    """What-if batched probe against a frozen state built by inserts."""
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import ClusterSim, Sizing, native_config
    from paper_2603_15202_b200 import _native
    trace, cfg = W.config1_chatbot()
    trace = trace.slice(300)
    h = _native.Handle(native_config(cfg, Sizing(1024, 4000)))
    h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
    refs = [OracleCache(None) for _ in range(cfg.n_instances)]
    rng = np.random.default_rng(3)
    for r in range(0, 300, 3):
        i = int(rng.integers(0, cfg.n_instances))
        a, b = int(trace.blk_off[r]), int(trace.blk_off[r + 1])
        keys = oracle_chain_keys(trace.blocks[a:b])
        cut = int(rng.integers(1, b - a + 1))
        h.cache_insert_keys(i, keys[:cut], r)
        refs[i].insert_keys(keys[:cut], r)
    got = h.probe_batch(0, 300)
    for r in range(300):
        a, b = int(trace.blk_off[r]), int(trace.blk_off[r + 1])
        keys = oracle_chain_keys(trace.blocks[a:b])
        want = [refs[i].match_keys(keys) for i in range(cfg.n_instances)]
        assert list(got[r]) == want, r
    h.close()


@pytest.mark.parametrize("builder", ["chat", "agent"])
def test_probe_batch_large_cluster_matches_oracle_cache(native, builder):
    """The block-per-request what-if probe of clusters >= 256 instances (depth-0 filter, then the
    two-stage probe for prompts <= 128 blocks or the deep warp probe beyond) against oracle caches:
    most instances hold nothing, some a partial chain, a few the whole chain."""
    import dataclasses
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import Sizing, native_config
    from paper_2603_15202_b200 import _native
    trace, cfg = W.chat_cluster(300, 400) if builder == "chat" else W.config3_agent(200, n_instances=300)
    cfg = dataclasses.replace(cfg, cache=dataclasses.replace(cfg.cache, capacity_blocks=None))
    n = 120
    trace = trace.slice(n)
    h = _native.Handle(native_config(cfg, Sizing(1024, 40000)))
    h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
    refs = {}
    rng = np.random.default_rng(5)
    for r in range(n):
        for i in rng.choice(cfg.n_instances, size=int(rng.integers(1, 6)), replace=False):
            a, b = int(trace.blk_off[r]), int(trace.blk_off[r + 1])
            keys = oracle_chain_keys(trace.blocks[a:b])
            cut = int(rng.integers(1, b - a + 1)) if rng.random() < 0.7 else b - a
            h.cache_insert_keys(int(i), keys[:cut], r)
            refs.setdefault(int(i), OracleCache(None)).insert_keys(keys[:cut], r)
    got = h.probe_batch(0, n)
    for r in range(n):
        a, b = int(trace.blk_off[r]), int(trace.blk_off[r + 1])
        keys = oracle_chain_keys(trace.blocks[a:b])
        want = [refs[i].match_keys(keys) if i in refs else 0 for i in range(cfg.n_instances)]
        assert list(got[r]) == want, r
    if builder == "agent":
        assert int(np.diff(trace.blk_off).max()) > 128       # the deep path ran
    h.close()


_ROUTE_POLICIES = ("simulate", "simulate_mistuned", "multiplicative", "vllm", "linear", "filter")


@pytest.mark.parametrize("name", _ROUTE_POLICIES)
def test_route_api_sequence_matches_reference(native, name):
    """ClusterSim.route on 80 consecutive records (queues grow, no steps) vs the reference's
    chosen instance and per-candidate scores (tests/golden/route_api.json,
    tools/make_route_golden.py)."""
    import json
    import os
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import ClusterConfig, CostModel, PolicyConfig
    want = json.load(open(os.path.join(G.GOLDEN, "route_api.json")))[name]
    pol = {"simulate": PolicyConfig(kind="simulate"),
           "simulate_mistuned": PolicyConfig(kind="simulate", mis_tuned=True, mis_tuned_factor=2.5),
           "multiplicative": PolicyConfig(), "vllm": PolicyConfig(kind="vllm", q_weight=0.5),
           "linear": PolicyConfig(kind="linear"), "filter": PolicyConfig(kind="filter", range_threshold=2)}[name]
    cfg = ClusterConfig(n_instances=5, cost_model=CostModel(chunk_tokens=256, max_batch_requests=6), policy=pol, seed=3)
    trace = W.config1_chatbot()[0].slice(80)
    sim = ClusterSim(cfg)
    for r, rec in enumerate(trace.records()):
        d = sim.route(rec, int(trace.arrival_us[r]))
        assert d.chosen == want[r][0], f"request {r}"
        assert [d.scores.get(i) for i in range(5)] == want[r][1], f"request {r}"
    sim.close()


@pytest.mark.parametrize("name", ["multiplicative", "vllm", "linear"])
def test_route_api_sequence_three_launch_path(native, name, monkeypatch):
    """The same route() sequences through the three-launch path (ingest, one-decision replay
    launch, output) that large shards and the extended kernel use, instead of route_kernel."""
    monkeypatch.setenv("RSIM_ROUTE_3LAUNCH", "1")
    test_route_api_sequence_matches_reference(native, name)


@pytest.mark.parametrize("kind,seed", [("simulate", 0), ("simulate", 1), ("filter", 0), ("filter", 1), ("filter", 2),
                                       ("linear", 0), ("linear", 1), ("linear", 2)])
def test_random_detector_simulate_match_oracle(native, kind, seed):
    """The hotspot detector steering the simulate policy (TTFT replay scores) and the filter
    policy (route_filter over the kept candidates): random hotspot traces and detector settings
    vs the oracle (pinned by the det_simulate_* / det_filter_* fixtures)."""
    import dataclasses
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import run
    from paper_2603_15202_b200.config import CacheConfig, DetectorConfig, PolicyConfig
    rng = np.random.default_rng(900 + seed + {"simulate": 0, "filter": 50, "linear": 70}[kind])
    for trial in range(3):
        N = int(rng.choice([3, 8, 16, 40]))
        trace, cfg = W.hotspot(N, int(rng.integers(300, 1200)), float(rng.uniform(0.4, 0.9)),
                               float(rng.uniform(20, 150)), int(rng.integers(1, 8)), seed=int(rng.integers(0, 99)))
        det = DetectorConfig(window_s=float(rng.choice([0.5, 1.0, 2.5, 7.0])), top_k_classes=int(rng.integers(1, 5)),
                             class_key_blocks=int(rng.integers(1, 3)),
                             consecutive_multiplier=float(rng.choice([0.0, 0.5, 1.0])),
                             mitigation=str(rng.choice(["exclude_holders", "force_least_bs"])),
                             compare_mean_non_holder=bool(rng.integers(0, 2)))
        pol = PolicyConfig(kind=kind, mis_tuned=bool(rng.integers(0, 2)), tie_break_seed=int(rng.integers(0, 9)),
                           range_threshold=int(rng.choice([1, 2, 4])))
        cap = [None, int(rng.integers(200, 2000))][int(rng.integers(0, 2))]
        cfg = dataclasses.replace(cfg, policy=pol, detector=det, cache=CacheConfig(16, cap))
        ref = run_oracle(trace, cfg)
        rep = run(trace, cfg)
        tag = f"seed{seed}/trial{trial} N={N} {det}"
        assert np.array_equal(rep.chosen, ref.chosen), tag
        rows = [(r.window_start_s, r.class_key, r.fraction, r.n_holders, r.n_others, r.suspect, r.phase)
                for r in rep.detector_rows]
        assert rows == ref.detector_rows, tag
