"""Diagnostic: replay every golden case on the GPU and report parity per case."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_cases as G  # noqa: E402
from paper_2603_15202_b200.cluster import run  # noqa: E402

fast = '--fast' in sys.argv
only = [a for a in sys.argv[1:] if not a.startswith('--')]
for name in G.names():
    if only and name not in only:
        continue
    if fast and name == 'cfg3_agent_evict_n16':
        continue
    tr, cfg = G.build(name)
    want = G.expected(name)
    t0 = time.time()
    try:
        rep = run(tr, cfg)
    except Exception as e:  # report and continue
        print(f"{name:28s} EXC {type(e).__name__}: {e}", flush=True)
        continue
    dt = time.time() - t0
    c = rep.columns
    bad = []
    for key in ("chosen", "hit_tokens", "first_sched_us", "first_token_us", "finish_us"):
        w = want[key]
        g = c[key]
        if not np.array_equal(g, w):
            i = int(np.nonzero(g != w)[0][0])
            bad.append(f"{key}@{i}(got {g[i]} want {w[i]})")
    steps = np.asarray([(s.instance, s.start_us, s.end_us, s.prefill_us) for s in rep.steps], np.int64).reshape(-1, 4)
    if not np.array_equal(steps, want["steps"]):
        bad.append(f"steps({len(steps)} vs {len(want['steps'])})")
    s = want["summary"]
    if (rep.end_us, rep.queued_at_last_arrival, rep.finished) != (s[0], s[1], s[2]):
        bad.append(f"summary {(rep.end_us, rep.queued_at_last_arrival, rep.finished)} vs {tuple(s[:3])}")
    print(f"{name:28s} R={len(tr):6d} {'OK ' if not bad else 'BAD'} {dt:7.2f}s {' '.join(bad[:3])}", flush=True)
