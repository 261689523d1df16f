"""Golden route-API sequences: the REFERENCE's ClusterSim.route (cluster.py:130-154) called
on consecutive records (no engine steps in between, so queues grow), recording the chosen
instance and every candidate's score, per policy.

    python tools/make_route_golden.py      # writes tests/golden/route_api.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refcompat import import_reference, to_ref_config, to_ref_records  # noqa: E402

from paper_2603_15202_b200 import workloads as W  # noqa: E402
from paper_2603_15202_b200.config import ClusterConfig, CostModel, PolicyConfig  # noqa: E402

POLICIES = {
    "simulate": PolicyConfig(kind="simulate"),
    "simulate_mistuned": PolicyConfig(kind="simulate", mis_tuned=True, mis_tuned_factor=2.5),
    "multiplicative": PolicyConfig(),
    "vllm": PolicyConfig(kind="vllm", q_weight=0.5),
    "linear": PolicyConfig(kind="linear"),
    "filter": PolicyConfig(kind="filter", range_threshold=2),
}


def main():
    rs = import_reference()
    from routesim.cluster import ClusterSim
    trace = W.config1_chatbot()[0].slice(80)
    out = {}
    for name, pol in POLICIES.items():
        cfg = ClusterConfig(n_instances=5, cost_model=CostModel(chunk_tokens=256, max_batch_requests=6), policy=pol, seed=3)
        sim = ClusterSim(to_ref_config(cfg))
        rows = []
        for r, rec in zip(range(len(trace)), to_ref_records(trace)):
            d = sim.route(rec, int(trace.arrival_us[r]))
            rows.append([d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)]])
        out[name] = rows
        print(name, [r[0] for r in rows[:20]])
    with open(os.path.join(ROOT, "tests", "golden", "route_api.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
