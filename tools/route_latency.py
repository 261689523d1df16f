"""Per-call latency of the online route() API vs the reference's (bench.measure_route_api).

    python tools/route_latency.py [workload:calls ...]     # default api64:2000 chat1024:500 chat16:2000
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

for spec in (sys.argv[1:] or ["chat16:2000", "api64:2000", "chat1024:500"]):
    name, n = spec.split(":")
    print(json.dumps(bench.measure_route_api(name, int(n), 0, with_ref=True)), flush=True)
