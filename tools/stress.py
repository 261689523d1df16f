"""Stress: replay golden cases repeatedly, checking chosen each time (hang/race hunting).
usage: python tools/stress.py REPEATS case [case ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_cases as G  # noqa: E402
from paper_2603_15202_b200.cluster import run  # noqa: E402

reps = int(sys.argv[1])
cases = sys.argv[2:] or [n for n in G.names() if n.startswith("det_")]
built = {n: (G.build(n), G.expected(n)) for n in cases}
for i in range(reps):
    for n, ((tr, cfg), want) in built.items():
        t0 = time.time()
        print(f"rep {i} {n} ...", end="", flush=True)
        rep = run(tr, cfg)
        ok = np.array_equal(rep.columns["chosen"], want["chosen"])
        print(f" {'ok' if ok else 'MISMATCH'} {time.time()-t0:.2f}s", flush=True)
