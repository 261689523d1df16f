"""Where a route() call's time goes: ctypes no-op, the C call alone, the kernel (CUDA events), and
a bare launch+sync round trip for comparison.   python tools/route_overhead.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200 import _native  # noqa: E402
from paper_2603_15202_b200.cluster import native_config, sizing_for  # noqa: E402


def p50(f, n=2000):
    ns = []
    for _ in range(n):
        t0 = time.perf_counter_ns()
        f()
        ns.append(time.perf_counter_ns() - t0)
    return float(np.percentile(np.asarray(ns) / 1e3, 50))


import torch  # noqa: E402
x = torch.zeros(16, device="cuda")
print("torch tiny kernel + synchronize:", round(p50(lambda: (x.add_(1), torch.cuda.synchronize())), 1), "us")
for name in ("chat16", "api64", "chat1024"):
    trace, cfg = bench.build_workload(name)
    n = 2000
    recs = trace.slice(n).records()
    h = _native.Handle(native_config(cfg, sizing_for(trace.slice(n), cfg), device=0))
    L = h._L
    print(name, "ctypes no-op (rsim_launch_count):", round(p50(lambda: L.rsim_launch_count(h._h)), 2), "us")
    blk = [np.asarray(r.prefix_blocks, np.uint64) for r in recs]
    it = iter(range(n))

    def one():
        i = next(it)
        r = recs[i]
        h.route_request(int(trace.arrival_us[i]), r.input_tokens, r.output_tokens, r.request_id, blk[i])
    print(name, "route_request (C ABI through the binding):", round(p50(one, n - 10), 1), "us")
    h.close()
