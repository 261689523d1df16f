"""Golden values of the reference's probe_capacity (cluster.py:295-330), run in this container.

    python tools/make_probe_golden.py     # writes tests/golden/probe_capacity.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refcompat import import_reference, to_ref_config, to_ref_records  # noqa: E402
from make_golden import build_case  # noqa: E402

CASES = {
    "chat_n4_mb4": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=4, cost_model=CostModel(max_batch_requests=4), seed=0))", 600, {}),
    "chat_n8_mb16": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=8, cost_model=CostModel(max_batch_requests=16), seed=1))", 800,
                     {"hi_start": 2.0, "iterations": 6}),
    "api_n4_vllm_mb8": ("(W.config2_api()[0], ClusterConfig(n_instances=4, cost_model=CostModel(max_batch_requests=8), policy=PolicyConfig(kind='vllm'), seed=2))", 600, {}),
    "chat_n3_simulate": ("(W.config1_chatbot()[0], ClusterConfig(n_instances=3, cost_model=CostModel(max_batch_requests=8), policy=PolicyConfig(kind='simulate'), seed=3))", 500,
                         {"hi_start": 4.0, "rate_cap": 64.0, "iterations": 5}),
}


def main():
    rs = import_reference()
    out = {}
    for name, (expr, prefix, kw) in CASES.items():
        trace, cfg = build_case(expr, prefix)
        t0 = time.perf_counter()
        v = rs.probe_capacity(to_ref_records(trace), to_ref_config(cfg), **kw)
        out[name] = {"expr": expr, "prefix": prefix, "kwargs": kw, "capacity_rps": v,
                     "reference_seconds": round(time.perf_counter() - t0, 2)}
        print(name, v, out[name]["reference_seconds"], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "probe_capacity.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
