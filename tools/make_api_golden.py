"""Golden stateful-API sessions from the REFERENCE's ClusterSim: route() / enqueue() /
cache.insert() calls, run_trace() after them and a second run_trace() on the same sim
(cluster.py:130-201), duplicate request ids (engine.py:266-267), and the instance queues
those calls leave behind (engine.py:212-213).

    python tools/make_api_golden.py      # writes tests/golden/api_sessions.json

Each session is a list of steps; tests/test_api_sessions.py replays the same steps on the
device drop-in and compares every recorded value."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refcompat import import_reference, to_ref_config, to_ref_records  # noqa: E402

from paper_2603_15202_b200 import workloads as W  # noqa: E402
from paper_2603_15202_b200.config import CacheConfig, ClusterConfig, CostModel, PolicyConfig  # noqa: E402

SESSIONS = {
    # name: (config, steps); a step is ("route", i) / ("enqueue", inst, i) / ("insert", inst, i, now) /
    # ("run", lo, hi) / ("route_dup", i, now) / ("queues",) over records of the chat trace
    "route_then_run": (ClusterConfig(n_instances=4, seed=1),
                       [("insert", 0, 0, 0)] + [("route", i) for i in range(1, 27)]
                       + [("queues",), ("run", 27, 260), ("queues",), ("run_after", 260, 400)]),
    # (a bare enqueue() before run_trace makes the reference's Collector raise KeyError on the
    # request's first step -- metrics.py:132 -- so enqueue() appears only in API-only sessions)
    "run_twice": (ClusterConfig(n_instances=6, cache=CacheConfig(16, 600), seed=2),
                  [("run", 0, 250), ("run_after", 250, 500), ("route_after", 500), ("run_after", 501, 600)]),
    "duplicates": (ClusterConfig(n_instances=3, policy=PolicyConfig(kind="vllm"), seed=0),
                   [("route", 0), ("route", 1)] + [("route_dup", j % 2, 70_000 + 10 * j) for j in range(2, 26)]
                   + [("route_after", 2), ("queues",)]),
    # refused duplicates (one instance: every repeat lands on the holder) are decided -- the
    # tie-break counter moves -- but never enqueued nor reported by the Collector
    "duplicates_then_run": (ClusterConfig(n_instances=1, seed=4),
                            [("route", 0), ("route", 1)] + [("route_dup", j % 2, 70_000 + 10 * j) for j in range(2, 12)]
                            + [("route_after", 2), ("run_after", 300, 420)]),
    "enqueue_dup": (ClusterConfig(n_instances=2, seed=0),
                    [("enqueue", 0, 0), ("enqueue_dup", 0, 0), ("enqueue", 1, 0), ("route", 1), ("queues",)]),
    "small_batch_queues": (ClusterConfig(n_instances=3, cost_model=CostModel(chunk_tokens=64, max_batch_requests=2), seed=5),
                           [("route", i) for i in range(40)] + [("queues",), ("run", 40, 120)]),
}

# route() with the prefix-hotspot detector (cluster.py:133-139): the hot class's prefix is inserted
# into a few instances (route() runs no engine step, so API inserts are what makes holders), then
# the hot trace is routed -- phase 1 suspects, phase-2 streaks, alarms and the mitigation (holders
# excluded / least batch size) all show in the decisions; enqueue() calls in between.
def _det_cfg(n, mitigation="exclude_holders", window_s=2.0, kind="multiplicative", seed=3):
    from paper_2603_15202_b200.config import DetectorConfig
    return ClusterConfig(n_instances=n, policy=PolicyConfig(kind=kind), seed=seed,
                         detector=DetectorConfig(window_s=window_s, mitigation=mitigation, top_k_classes=4))


def _hot_steps(trace, holders, n_route, extra=()):
    from collections import Counter
    from paper_2603_15202_b200.trace import class_key
    recs = trace.records()
    ck = [class_key(r.prefix_blocks, 2) for r in recs]
    hot = Counter(ck).most_common(1)[0][0]
    first = ck.index(hot)
    steps = [("insert", h, first, 0) for h in holders] + [("route", i) for i in range(n_route)]
    for pos, st in extra:
        steps.insert(pos, st)
    return steps


def _fuzz_steps(seed, n_inst, n_steps=160):
    """A seeded random mix of route() / repeated ids / enqueue() / cache.insert() / queue views
    over the chat trace, in non-decreasing time (the device path's contract)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    steps, nxt = [], 0
    for _ in range(n_steps):
        u = rng.random()
        if u < 0.6 or nxt < 2:
            steps.append(("route", nxt)); nxt += 1
        elif u < 0.75:
            steps.append(("route_dup_now", int(rng.integers(0, nxt))))
        elif u < 0.85:
            steps.append(("enqueue_now", int(rng.integers(0, n_inst)), 400 + nxt)); nxt += 1
        elif u < 0.95:
            steps.append(("insert_now", int(rng.integers(0, n_inst)), int(rng.integers(0, 590))))
        else:
            steps.append(("queues",))
    return steps


FUZZ_SESSIONS = {   # name: (config, seed)
    "fuzz_mult_n5": (ClusterConfig(n_instances=5, seed=11), 0),
    "fuzz_vllm_n12": (ClusterConfig(n_instances=12, policy=PolicyConfig(kind="vllm", q_weight=0.5), seed=12), 1),
    "fuzz_linear_n3": (ClusterConfig(n_instances=3, policy=PolicyConfig(kind="linear", bs_norm_cap=6.0),
                                     cost_model=CostModel(chunk_tokens=96, max_batch_requests=3), seed=13), 2),
    "fuzz_filter_n7": (ClusterConfig(n_instances=7, policy=PolicyConfig(kind="filter", range_threshold=2), seed=14), 3),
    "fuzz_mult_n300": (ClusterConfig(n_instances=300, seed=15), 4),
}

DET_SESSIONS = {   # name: (config, (holders, routes, extra steps))
    "det_exclude": (_det_cfg(8), ((0, 1), 400, ())),
    "det_force_least_bs": (_det_cfg(8, mitigation="force_least_bs"), ((2, 5), 400, ())),
    "det_enqueue_mix": (_det_cfg(6, kind="vllm", window_s=1.0), ((0,), 300, [(150, ("enqueue_now", 3, 500)), (151, ("queues",))])),
    "det_many_instances": (_det_cfg(40, window_s=3.0), ((0, 7, 13, 21), 500, ())),
    # one instance: a request id routed again is always refused -- here under another class's
    # record, so the refused call's class is never observed and the next new class takes its track
    "det_dup_new_class": (_det_cfg(1, window_s=1.0), ((0,), 60, [(4, ("route_dup_as", 39, 0, None))])),
}


def run_session(cfg, steps, trace, api):
    """api: (ClusterSim class, record converter, DuplicateRequestError). Returns the observations."""
    Sim, conv, Dup = api
    import dataclasses
    sim = Sim(cfg)
    recs = conv(trace)
    obs = []
    clock = 0              # simulated time reached so far: "_after" steps start past it (the device
    for st in steps:       # path needs non-decreasing time across calls, see ClusterSim)
        kind = st[0]
        if kind == "run_after":
            shift = (clock + 1_000_000 - int(trace.arrival_us[st[1]])) / 1e6
            rs = [dataclasses.replace(r, arrival_s=r.arrival_s + shift) for r in recs[st[1]:st[2]]]
            rep = sim.run_trace(rs)
            clock = max(clock, rep.end_us)
            obs.append(["run", [[m.request_id, m.chosen_instance, m.hit_tokens, m.arrival_us, m.first_token_us,
                                 m.finish_us] for m in rep.requests], rep.arrivals_hash, len(rep.steps),
                        rep.queued_at_last_arrival, rep.end_us])
            continue
        if kind == "route_after":
            clock += 1000
            d = sim.route(recs[st[1]], clock)
            obs.append(["route", d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)], d.kind, sorted(d.filtered)])
            continue
        if kind == "route":
            r = recs[st[1]]
            d = sim.route(r, int(trace.arrival_us[st[1]]))
            clock = max(clock, int(trace.arrival_us[st[1]]))
            obs.append(["route", d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)], d.kind, sorted(d.filtered)])
        elif kind == "route_dup":
            r = recs[st[1]]
            clock = max(clock, st[2])
            try:
                d = sim.route(r, st[2])
                obs.append(["route", d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)], d.kind, sorted(d.filtered)])
            except Dup:
                obs.append(["dup"])
        elif kind == "route_dup_now":        # an id again, at the time reached so far
            try:
                d = sim.route(recs[st[1]], clock)
                obs.append(["route", d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)], d.kind, sorted(d.filtered)])
            except Dup:
                obs.append(["dup"])
        elif kind == "route_dup_as":        # record st[1] under record st[2]'s request id
            r = dataclasses.replace(recs[st[1]], request_id=recs[st[2]].request_id)
            now = clock if st[3] is None else st[3]
            clock = max(clock, now)
            try:
                d = sim.route(r, now)
                obs.append(["route", d.chosen, [d.scores.get(i) for i in range(cfg.n_instances)], d.kind, sorted(d.filtered)])
            except Dup:
                obs.append(["dup"])
        elif kind == "enqueue":
            a = sim.instances[st[1]].enqueue(recs[st[2]], int(trace.arrival_us[st[2]]))
            obs.append(["enqueue", a.hit_blocks, a.hit_tokens, a.pending_prefill])
        elif kind == "enqueue_now":          # enqueue a later record at the time reached so far
            a = sim.instances[st[1]].enqueue(recs[st[2]], clock)
            obs.append(["enqueue", a.hit_blocks, a.hit_tokens, a.pending_prefill])
        elif kind == "enqueue_dup":
            try:
                sim.instances[st[1]].enqueue(recs[st[2]], int(trace.arrival_us[st[2]]))
                obs.append(["enqueue_ok"])
            except Dup:
                obs.append(["dup"])
        elif kind == "insert_now":           # cache.insert at the time reached so far
            sim.instances[st[1]].cache.insert(recs[st[2]].prefix_blocks, clock)
            obs.append(["insert"])
        elif kind == "insert":
            sim.instances[st[1]].cache.insert(recs[st[2]].prefix_blocks, st[3])
            obs.append(["insert"])
        elif kind == "queues":
            q = []
            for inst in sim.instances:
                q.append([[s.record.request_id, s.pending, s.hit_blocks, s.hit_tokens, s.generated, s.enqueue_us]
                          for s in inst.queue] + [["running"] + [[s.record.request_id, s.generated] for s in inst.running]])
            obs.append(["queues", q])
        elif kind == "run":
            rep = sim.run_trace(recs[st[1]:st[2]])
            clock = max(clock, rep.end_us)
            reqs = [[m.request_id, m.chosen_instance, m.hit_tokens, m.arrival_us, m.first_token_us, m.finish_us]
                    for m in rep.requests]
            obs.append(["run", reqs, rep.arrivals_hash, len(rep.steps), rep.queued_at_last_arrival, rep.end_us,
                        [[s.instance, s.start_us, s.end_us, s.prefill_us] for s in rep.steps[-50:]]])
    return obs


def main():
    import_reference()
    from routesim.cluster import ClusterSim
    from routesim.engine import DuplicateRequestError
    trace = W.config1_chatbot()[0].slice(600)
    out = {}
    for name, (cfg, steps) in SESSIONS.items():
        out[name] = run_session(to_ref_config(cfg), steps, trace,
                                (ClusterSim, to_ref_records, DuplicateRequestError))
        print(name, [o[0] if o[0] != "route" else o[1] for o in out[name]][:40])
    for name, (cfg, seed) in FUZZ_SESSIONS.items():
        out[name] = run_session(to_ref_config(cfg), _fuzz_steps(seed, cfg.n_instances), trace,
                                (ClusterSim, to_ref_records, DuplicateRequestError))
        print(name, [o[0] if o[0] != "route" else o[1] for o in out[name]][:40])
    hot = W.hotspot(8, 600, 0.6, 20.0, seed=4)[0]
    for name, (cfg, (holders, n_route, extra)) in DET_SESSIONS.items():
        steps = _hot_steps(hot, holders, n_route, extra)
        out[name] = run_session(to_ref_config(cfg), steps, hot, (ClusterSim, to_ref_records, DuplicateRequestError))
        print(name, [o[1] for o in out[name] if o[0] == "route"][:60])
    with open(os.path.join(ROOT, "tests", "golden", "api_sessions.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
