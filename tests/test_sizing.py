"""Host sizing of the per-instance KV$ tables (CPU): sized from the estimated DISTINCT keys an
instance ends up holding, so the tables of a large cluster stay L2-sized (VERDICT r1 weak #4:
sizing from the routed chain lengths made chat1024's tables 10x too large). Checked against the
real per-instance key sets of the oracle's replay (no eviction: the final table = the union of
the routed chains, kvcache.py:81-104)."""
import numpy as np
import pytest

from oracle.oracle import chain_keys, run_oracle


def _real_distinct(trace, cfg):
    ref = run_oracle(trace, cfg)
    bs = cfg.cache.block_size
    sets = [set() for _ in range(cfg.n_instances)]
    out = np.zeros(cfg.n_instances, np.int64)
    off = trace.blk_off
    outb = (trace.out_tokens + bs - 1) // bs
    for r in range(len(trace)):
        c = int(ref.chosen[r])
        sets[c].update(chain_keys(trace.blocks[off[r]:off[r + 1]]).tolist())
        out[c] += outb[r]
    return np.array([len(s) for s in sets]) + out


@pytest.mark.parametrize("builder", ["config1_chatbot()", "chat_cluster(256, 20_000)", "config2_api(20_000)"])
def test_table_sizing_fits_distinct_keys(builder):
    from paper_2603_15202_b200 import workloads as W
    from paper_2603_15202_b200.cluster import sizing_for
    trace, cfg = eval("W." + builder, {"W": W})
    real = _real_distinct(trace, cfg)
    sz = sizing_for(trace, cfg)
    slots = 1 << int(np.ceil(np.log2(sz.expected_keys * 4 / 3 + 64)))   # rsim_create's rounding
    assert real.max() <= 3 * slots // 4, (builder, real.max(), slots)    # no RSIM_E_TABLE_FULL regrow
    assert slots <= 4 * real.max(), (builder, real.max(), slots)         # and no 10x overshoot
