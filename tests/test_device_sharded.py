"""Sharded replay: the instances split over 2-4 ranks (handles sharing one
device, exchanging per-decision partials through device mailboxes) must make
exactly the decisions of the unsharded reference run."""
import numpy as np
import pytest

import golden_cases as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("adv_mixed_n33", 2), ("adv_mixed_n33", 3), ("cfg1_chatbot_full", 2),
                                        ("cfg2_api_prefix4000", 4), ("adv_same_time_ties", 4),
                                        ("evict_heavy_n4", 2), ("stale_50ms_n16", 3), ("stale_5ms", 2),
                                        ("policy_simulate_mistuned", 3), ("policy_simulate_agent_evict", 2),
                                        ("cfg1_chatbot_full", 8), ("adv_mixed_n33", 8), ("cfg2_api_prefix4000", 8),
                                        # route_filter across ranks: the batch-size range is global
                                        ("policy_filter", 2), ("policy_filter_r2", 3), ("policy_filter", 8),
                                        ("stale_filter_evict", 2),
                                        # linear without a cap: the per-decision bs max over every rank
                                        ("policy_linear", 2), ("policy_linear", 8), ("stale_linear", 3)])
def test_sharded_matches_reference(name, world):
    from paper_2603_15202_b200.distributed import run_sharded_local
    trace, cfg = G.build(name)
    want = G.expected(name)
    got = run_sharded_local(trace, cfg, world)
    for key in ("chosen", "hit_tokens", "first_sched_us", "first_token_us", "finish_us"):
        assert np.array_equal(got[key], want[key]), key


@pytest.mark.parametrize("name,world,n", [("adv_mixed_n33", 2, 120), ("cfg1_chatbot_full", 2, 150)])
def test_sharded_processes_match_reference(name, world, n):
    """One process per shard (torchrun), mailboxes shared through CUDA IPC handles."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tools", "sharded_check.py"), name, str(n)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "OK" in p.stdout


@pytest.mark.parametrize("world,seed", [(2, 0), (3, 1), (5, 2)])
def test_sharded_filter_random_matches_oracle(world, seed):
    """route_filter with the instances split over ranks: random clusters, thresholds and cost
    models (the range test flips between branches decision by decision) vs the oracle."""
    import dataclasses
    from oracle.oracle import run_oracle
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.config import CostModel, PolicyConfig
    from paper_2603_15202_b200.distributed import run_sharded_local
    rng = np.random.default_rng(700 + seed)
    N = int(rng.choice([5, 11, 24]))
    trace, cfg = W.chat_cluster(N, 1500, float(rng.uniform(1.0, 6.0)), seed=seed)
    cfg = dataclasses.replace(cfg, policy=PolicyConfig(kind="filter", range_threshold=int(rng.integers(0, 4))),
                              cost_model=CostModel(chunk_tokens=int(rng.choice([256, 2048])),
                                                   max_batch_requests=int(rng.choice([4, 256]))))
    got = run_sharded_local(trace, cfg, world)
    want = run_oracle(trace, cfg)
    assert np.array_equal(got["chosen"], want.chosen)
    assert np.array_equal(got["finish_us"], want.finish_us)
