"""Where the e2e (run(records, config)) time goes beyond the device replay: cProfile of one call.

    python tools/e2e_profile.py WORKLOAD
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200.cluster import run  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "agent256"
trace, cfg = bench.build_workload(name)
for _ in range(2):
    run(trace, cfg)
t0 = time.perf_counter()
rep = run(trace, cfg)
print(f"{name}: run() {1000 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
rep = run(trace, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
