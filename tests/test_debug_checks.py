"""ClusterConfig.debug_checks on the device: after every decision (its engine steps) and after
the drain, InstanceSim.reconcile (engine.py:248-258) and PrefixCache.check_invariants
(kvcache.py:178-194) run over every instance (csrc/rsim_check.cuh). Correct replays pass them
with unchanged decisions; injected faults raise InvariantError naming the failed check."""
import dataclasses

import numpy as np
import pytest

import golden_cases as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n", [("cfg1_chatbot_full", 1500), ("evict_heavy_n4", None), ("adv_tight_capacity", None),
                                    ("stale_5ms", 800), ("policy_simulate_agent_evict", 300),
                                    ("adv_out1", None), ("cost_small_batch", None)])
def test_debug_replay_passes_and_matches(name, n):
    from paper_2603_15202_b200.cluster import run
    trace, cfg = G.build(name)
    if n is not None:
        trace = trace.slice(min(n, len(trace)))
    want = G.expected(name)
    rep = run(trace, dataclasses.replace(cfg, debug_checks=True))
    k = len(trace)
    assert np.array_equal(rep.chosen, want["chosen"][:k])
    assert np.array_equal(rep.hit_tokens, want["hit_tokens"][:k])
    # finish times of a prefix depend on the requests it drops: compare with the oracle's prefix run
    from oracle.oracle import run_oracle
    assert np.array_equal(rep.columns["finish_us"], run_oracle(trace, cfg).finish_us)


@pytest.mark.parametrize("what,text", [(0, "pin must cover the path"), (1, "reconcile"),
                                       (2, "parent older than child")])
def test_injected_fault_is_reported(what, text):
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import InvariantError
    trace, cfg = G.build("evict_heavy_n4")
    trace = trace.slice(200)
    sim = ClusterSim(dataclasses.replace(cfg, debug_checks=True))
    h = sim._device()
    h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
    h.replay(0, 120)                     # mid-trace: queued and running requests, pinned chains
    h.check_invariants()
    occ = h.instances()[:, 11]
    inst = int(np.argmax(occ))
    h.debug_corrupt(inst, what)
    with pytest.raises(InvariantError, match=text):
        h.check_invariants()
    sim.close()


def test_api_inserts_are_covered():
    """Chains inserted through the PrefixCache API are walked too (no orphan reports)."""
    from paper_2603_15202_b200.cluster import ClusterSim
    from paper_2603_15202_b200.config import CacheConfig, ClusterConfig
    sim = ClusterSim(ClusterConfig(n_instances=2, cache=CacheConfig(16, 40), debug_checks=True))
    rng = np.random.default_rng(0)
    for i in range(60):
        sim.instances[i % 2].cache.insert([int(x) for x in rng.integers(1, 4, size=int(rng.integers(1, 12)))], i)
    sim._device().check_invariants()
    sim.close()
