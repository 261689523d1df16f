"""A short route()-API session for launch-list profiling: python tools/route_launches.py WORKLOAD CALLS"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200 import _native  # noqa: E402
from paper_2603_15202_b200.cluster import native_config, sizing_for  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
trace, cfg = bench.build_workload(name)
recs = trace.slice(n).records()
h = _native.Handle(native_config(cfg, sizing_for(trace.slice(n), cfg), device=0))
ns = []
for r, t in zip(recs, trace.arrival_us[:n]):
    b = np.asarray(r.prefix_blocks, np.uint64)
    t0 = time.perf_counter_ns()
    h.route_request(int(t), r.input_tokens, r.output_tokens, r.request_id, b)
    ns.append(time.perf_counter_ns() - t0)
print(name, "p50 us", np.percentile(np.asarray(ns) / 1e3, 50))
