"""Pin the CPU oracle to the reference: every golden fixture and hash KAT."""
import numpy as np
import pytest

import golden_cases as G
from oracle.oracle import OracleCache, chain_keys, run_oracle
from paper_2603_15202_b200 import hashing


def test_hash_kats_host_and_oracle():
    k = G.kats()
    for v, want in k["splitmix64"]:
        assert hashing.splitmix64(v) == want
    for a, b, want in k["combine64"]:
        assert hashing.combine64(a, b) == want
    for vals, want in k["stable_key"]:
        assert hashing.stable_key(*vals) == want
        assert int(np.asarray(hashing.stable_key_np(*vals))) == want
    for blocks, want in k["chain_keys"]:
        assert hashing.chain_keys(blocks) == want
        assert [int(x) for x in chain_keys(blocks)] == want
    from paper_2603_15202_b200.trace import class_key
    for blocks, want in k["class_key"]:
        assert class_key(blocks) == want


@pytest.mark.parametrize("name", G.names())
def test_oracle_matches_reference(name):
    trace, cfg = G.build(name)
    want = G.expected(name)
    got = run_oracle(trace, cfg, with_log=True)
    assert np.array_equal(got.chosen, want["chosen"])
    assert np.array_equal(got.hit_tokens, want["hit_tokens"])
    assert np.array_equal(got.first_sched_us, want["first_sched_us"])
    assert np.array_equal(got.first_token_us, want["first_token_us"])
    assert np.array_equal(got.finish_us, want["finish_us"])
    steps = got.log[got.log[:, 0] == 1][:, [1, 2, 3, 4]]
    assert np.array_equal(steps, want["steps"])
    s = want["summary"]
    assert (got.end_us, got.queued_at_last_arrival, got.finished) == (s[0], s[1], s[2])
    if "det_ints" in want:                         # detector.finalize rows + first violation
        assert got.detector_rows == G.detector_rows(want)
        assert got.first_violation_us == G.first_violation(want)


def test_oracle_cache_lru_examples():
    # reference test_kvcache.py:39-49 and :65-75
    c = OracleCache(4)
    c.insert_keys(chain_keys([101, 102, 103, 104]), 0)
    assert c.insert_keys(chain_keys([201, 202]), 10) == 2
    assert c.match_keys(chain_keys([101, 102, 103, 104])) == 2
    c = OracleCache(4)
    c.insert_keys(chain_keys([1, 2]), 0)
    c.insert_keys(chain_keys([11, 12]), 1)
    k = chain_keys([1, 2])
    c.touch_keys(k, c.match_keys(k), 2)
    c.insert_keys(chain_keys([21, 22]), 3)
    assert c.match_keys(chain_keys([1, 2])) == 2 and c.match_keys(chain_keys([11, 12])) == 0


def test_oracle_detector_empty_prefix_raises():
    """class_key of an empty prefix raises ValueError (reference detector.py:43-44)."""
    import dataclasses
    from paper_2603_15202_b200.config import DetectorConfig
    trace, cfg = G.build("adv_zero_bs")
    import numpy as np
    from paper_2603_15202_b200.trace import PackedTrace
    t = PackedTrace(trace.request_id[:2], trace.arrival_s[:2], trace.in_tokens[:2], trace.out_tokens[:2],
                    trace.class_key[:2], np.zeros(3, np.int64), np.zeros(0, np.uint64))
    with pytest.raises(ValueError):
        run_oracle(t, dataclasses.replace(cfg, detector=DetectorConfig()))
