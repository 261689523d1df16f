"""Sharded replay: the instances split over 2-4 ranks (handles sharing one
device, exchanging per-decision partials through device mailboxes) must make
exactly the decisions of the unsharded reference run."""
import numpy as np
import pytest

import golden_cases as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world", [("adv_mixed_n33", 2), ("adv_mixed_n33", 3), ("cfg1_chatbot_full", 2),
                                        ("cfg2_api_prefix4000", 4), ("adv_same_time_ties", 4),
                                        ("evict_heavy_n4", 2)])
def test_sharded_matches_reference(name, world):
    from paper_2603_15202_b200.distributed import run_sharded_local
    trace, cfg = G.build(name)
    want = G.expected(name)
    got = run_sharded_local(trace, cfg, world)
    for key in ("chosen", "hit_tokens", "first_sched_us", "first_token_us", "finish_us"):
        assert np.array_equal(got[key], want[key]), key
