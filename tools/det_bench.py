"""Replay time with and without the hotspot detector on a hotspot trace.

    python tools/det_bench.py [n_instances] [n_requests]
"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_15202_b200 import workloads as W  # noqa: E402
from paper_2603_15202_b200.cluster import ClusterSim  # noqa: E402
from paper_2603_15202_b200.config import DetectorConfig  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
trace, cfg = W.hotspot(N, R, 0.6, 40.0 * N / 16)
for det, kw in ((None, {}), (None, {"ctas": 1}), (DetectorConfig(window_s=5.0), {})):
    c = dataclasses.replace(cfg, detector=det)
    sim = ClusterSim(c, **kw)
    rep = sim.run_trace(trace)
    h = sim._handle
    best = min(h.rerun() for _ in range(3))
    rows = len(rep.detector_rows)
    print(f"hotspot N={N} R={len(trace)} detector={'on' if det else 'off'} {kw or ''}: {best:.2f} ms "
          f"({1000 * best / len(trace):.2f} us/decision), rows {rows}", flush=True)
    sim.close()
