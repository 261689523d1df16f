"""cProfile of ClusterSim.route() on the GPU (the host-side share of a call):
python tools/route_pyprof.py [workload] [calls]"""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200.cluster import ClusterSim  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "chat1024"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
trace, cfg = bench.build_workload(name)
recs = trace.slice(n + 100).records()
sim = ClusterSim(cfg)
for i in range(100):
    sim.route(recs[i], int(trace.arrival_us[i]))
pr = cProfile.Profile()
pr.enable()
for i in range(100, 100 + n):
    sim.route(recs[i], int(trace.arrival_us[i]))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
