"""Per-decision latency outliers of a workload (commit-to-commit %globaltimer deltas)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200 import _native  # noqa: E402
from paper_2603_15202_b200.cluster import native_config, sizing_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "agent256"
trace, cfg = bench.build_workload(name)
h = _native.Handle(native_config(cfg, sizing_for(trace, cfg)))
h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
h.rerun()
R = len(trace)
ns = h.decision_ns(0, R)
lat = np.diff(ns) / 1000.0
B = np.diff(trace.blk_off)
print(f"{name}: p50 {np.percentile(lat, 50):.1f} p90 {np.percentile(lat, 90):.1f} p99 {np.percentile(lat, 99):.1f} "
      f"max {lat.max():.1f} us; share of time in decisions > 200 us: {lat[lat > 200].sum() / lat.sum():.2%}")
for q in (200, 500, 1000):
    print(f"  decisions > {q} us: {(lat > q).sum()}")
top = np.argsort(-lat)[:12]
for i in top:
    k = i + 1
    print(f"  k={k} lat {lat[i]:.0f} us  B={B[k]} in={trace.in_tokens[k]} out={trace.out_tokens[k]} dt_arrival_us={trace.arrival_us[k] - trace.arrival_us[k - 1]}")
h.close()
