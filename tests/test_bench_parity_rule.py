"""bench.py's prefix parity rule (CPU): against an oracle run over a prefix of the trace, every
decision is comparable, but a finish time only for requests that finish before the first
excluded arrival -- later arrivals join still-running batches (the full run of the same oracle
stands in for the device here)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_prefix_parity_compares_only_settled_finishes():
    import bench
    from oracle.oracle import run_oracle
    from paper_2603_15202_b200 import workloads as W
    trace, cfg = W.config1_chatbot()
    full = run_oracle(trace.slice(3000), cfg)
    pre = run_oracle(trace.slice(1000), cfg)
    naive = bench.parity_vs_oracle(pre, full.chosen, full.hit_tokens, full.finish_us, 3000)
    assert naive["by_field"]["chosen"] == 0 and naive["by_field"]["hit_tokens"] == 0
    assert naive["by_field"]["finish_us"] > 0            # in-flight requests at the cut moved
    ruled = bench.parity_vs_oracle(pre, full.chosen, full.hit_tokens, full.finish_us, 3000,
                                   bench._cutoff(trace.slice(3000), 1000))
    assert ruled["mismatches"] == 0 and 0 < ruled["finish_compared"] < 1000
    assert bench._cutoff(trace.slice(1000), 1000) is None
    bad = np.array(full.chosen, copy=True)
    bad[10] ^= 1
    assert bench.parity_vs_oracle(pre, bad, full.hit_tokens, full.finish_us, 3000, 0)["first_mismatch"] == 10
