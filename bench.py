#!/usr/bin/env python
"""Benchmark: routing decisions/s of the multiplicative router (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload api64|chat1024|...]
    python bench.py --impl reference ...        # the reference's own CPU scheduler

A *step* is one full replay of the workload trace: every routing decision
(chain hash, KV$ probe of every instance, multiplicative score, rotating
tie-break argmin, enqueue) plus every engine step and KV$ update between
arrivals, then the final drain -- exactly ``run(records, config)``.

* ``value``  : decisions/s with the trace resident in HBM (device time of
               reset + K1 + replay + drain, CUDA events on librsim's stream).
* ``e2e``    : decisions/s through the public API ``run(records, config)``
               with host numpy inputs: H2D of the trace, K1, replay, drain and
               D2H of every per-request result are inside the timed region.
* ``roofline``: the replay kernel's algorithmic bytes per launch
               over its CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline``: the reference (routesim, CPython, 1 core) on a bounded
               prefix sample of the same trace, timed on this host; the C
               oracle port over the full trace is reported beside it.

The trace and L2 working set are larger than the 126 MB L2 for api64 and the
replay rewrites the device tables every step; an explicit 512 MB L2 flush
is also done between timed steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (builder, description)
    "api64": ("config2_api()", "synthetic API-call trace, 32 shared 1024-token system prompts, 64 instances, ~100k requests (BASELINE configs[1])"),
    "chat1024": ("chat_cluster(1024, 100_000)", "synthetic chat trace (8 classes), 1024 instances at 3 req/s/instance, ~100k requests (north-star 1024-instance target)"),
    "chat16": ("config1_chatbot()", "synthetic chatbot trace, 16 instances, ~10k requests (BASELINE configs[0])"),
    "agent256": ("config3_agent(20_000)", "multi-turn coding-agent trace, 32k-token prompts, 256 instances, capacity 16384 (BASELINE configs[2])"),
    "large4096": ("config4_large(1_000_000)", "4096-instance chat cluster, ~1M requests (BASELINE configs[3])"),
    "adv64": ("adversarial_stream(64, 100_000)", "adversarial stream (N-way same-time ties, bs 0 vs 1, full hits, out = 1, ragged inputs, tight-capacity evictions), 64 instances, 100k requests (BASELINE configs[4])"),
    "hot64det": ("hotspot_detector(64, 20_000)", "prefix-hotspot trace (one class 60 % of arrivals), 64 instances, reference detector on (SURVEY 8f rank 1)"),
}
METRIC = "routing decisions/sec"


def build_workload(name: str):
    from paper_2603_15202_b200 import workloads as W
    return eval("W." + WORKLOADS[name][0], {"W": W})


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def flush_l2(dev):
    import torch
    buf = getattr(flush_l2, "_buf", None)
    if buf is None:
        buf = flush_l2._buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    buf.fill_(1)
    torch.cuda.synchronize(dev)


# ------------------------------------------------------------------------------ reference arm
def reference_samples(trace, cfg, budget_s: float):
    """Prefix length of the trace the reference replays in about ``budget_s``."""
    rate = 2400.0 * (16.0 / max(cfg.n_instances, 16)) ** 0.6   # CPython e2e decisions/s
    return min(len(trace), max(200, int(budget_s * rate)))


def import_reference():
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "routesim")):
        if path not in sys.path:
            sys.path.insert(0, path)
        import routesim  # noqa: F401
        return routesim
    return None


def ref_records_and_config(trace, cfg):
    import routesim
    from routesim.cluster import CacheConfig, ClusterConfig
    from routesim.engine import CostModel
    from routesim.policies import PolicyConfig
    from routesim.trace import TraceRecord
    cm = cfg.cost_model
    rcfg = ClusterConfig(n_instances=cfg.n_instances,
                         cost_model=CostModel(cm.prefill_base_ms, cm.prefill_per_token_ms, cm.decode_base_ms,
                                              cm.decode_per_seq_ms, cm.decode_per_ctx_token_ms, cm.chunk_tokens,
                                              cm.max_batch_requests),
                         cache=CacheConfig(cfg.cache.block_size, cfg.cache.capacity_blocks),
                         policy=PolicyConfig(**{k: getattr(cfg.policy, k) for k in cfg.policy.__dataclass_fields__}),
                         staleness_ms=cfg.staleness_ms, seed=cfg.seed,
                         detector=None if cfg.detector is None else __import__("routesim.detector", fromlist=["x"]).DetectorConfig(
                             **{k: getattr(cfg.detector, k) for k in cfg.detector.__dataclass_fields__}))
    recs = [TraceRecord(r.request_id, r.arrival_s, r.prefix_blocks, r.input_tokens, r.output_tokens, r.class_key)
            for r in trace.records()]
    return routesim, recs, rcfg


def time_reference(trace, cfg, n_sample: int, repeats: int = 1):
    """CPython reference ``routesim.run`` on the first n_sample records; best decisions/s."""
    rs = import_reference()
    if rs is None:
        return None
    sample = trace.slice(n_sample)
    routesim, recs, rcfg = ref_records_and_config(sample, cfg)
    best = 0.0
    for _ in range(repeats):
        t0 = time.perf_counter()
        routesim.run(recs, rcfg)
        dt = time.perf_counter() - t0
        best = max(best, len(recs) / dt)
    return best


def time_port(trace, cfg):
    """The C oracle port (oracle/rsim_oracle.c, 1 thread) over ``trace``: (decisions/s, result).
    The result is the parity checker of the device replay (parity_vs_oracle)."""
    from oracle.oracle import run_oracle
    t0 = time.perf_counter()
    res = run_oracle(trace, cfg)
    return len(trace) / (time.perf_counter() - t0), res


def parity_vs_oracle(ref, chosen, hit_tokens, finish_us, n_total, cutoff_us=None):
    """Decision-by-decision comparison of the device replay with the oracle (which is pinned to
    the reference's own run(), tests/golden): chosen instance and hit tokens of every request the
    oracle replayed (all of them, or a prefix: decision k depends only on records[:k+1], SURVEY
    8c), and the finish time of every request that finishes before ``cutoff_us``, the arrival of
    the first request outside the prefix (a later arrival can join a still-running request's
    batch and move its finish; None = the full trace, every finish compared)."""
    n = len(ref.chosen)
    fin = np.ones(n, bool) if cutoff_us is None else (np.asarray(ref.finish_us) < cutoff_us)
    bad_f = (ref.finish_us != finish_us[:n]) & fin
    mism = {"chosen": int((ref.chosen != chosen[:n]).sum()),
            "hit_tokens": int((ref.hit_tokens != hit_tokens[:n]).sum()),
            "finish_us": int(bad_f.sum())}
    first = None
    bad = (ref.chosen != chosen[:n]) | (ref.hit_tokens != hit_tokens[:n]) | bad_f
    if bad.any():
        first = int(np.argmax(bad))
    return {"vs": "oracle/rsim_oracle.c (pinned to the reference's run(), tests/golden)",
            "decisions": n, "of": n_total, "finish_compared": int(fin.sum()), "mismatches": sum(mism.values()),
            "by_field": mism, "first_mismatch": first, "evicted_blocks": int(getattr(ref, "evicted", 0))}


def _cutoff(trace, n):
    """Arrival (us) of the first request beyond a parity prefix of n requests (None: no prefix)."""
    return None if n >= len(trace) else int(trace.arrival_us[n])


def chosen_digest(chosen) -> str:
    """sha256 (first 16 hex) of the int32 decision log: equal across G = 1, 2, 4, 8."""
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(chosen, dtype=np.int32).tobytes()).hexdigest()[:16]


def host_cpu():
    """lscpu model name and the host's logical core count."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    trace, cfg = build_workload(args.workload)
    rs = import_reference()
    cores = 1
    if rs is not None:
        n = reference_samples(trace, cfg, args.ref_budget_s)
        routesim, recs, rcfg = ref_records_and_config(trace.slice(n), cfg)
        kind, sample = "reference", f"first {n} of {len(trace)} requests of {args.workload}, routesim.run (CPython, 1 thread)"
        run_step = lambda: routesim.run(recs, rcfg)  # noqa: E731
    else:
        from oracle.oracle import run_oracle
        n = len(trace)
        kind, sample = "port", f"all {n} requests of {args.workload}, C oracle port (1 thread)"
        run_step = lambda: run_oracle(trace, cfg)  # noqa: E731
    for _ in range(args.warmup):
        run_step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run_step()
        times.append(time.perf_counter() - t0)
    value = n * len(times) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": "decisions/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": args.workload, "description": WORKLOADS[args.workload][1],
                                            "n_instances": cfg.n_instances, "requests": n},
            "cpu_baseline": {"value": value, "unit": "decisions/s", "cores": cores, "kind": kind, "sample": sample,
                             "host_cpu": host_cpu()},
            "e2e": {"value": value, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ our arm
def measure_workload(name, args, dev_index, with_cpu: bool, rank: int):
    import torch
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.cluster import native_config, release_pool, run, sizing_for

    trace, cfg = build_workload(name)
    R = len(trace)
    dev = torch.device("cuda", dev_index)
    # resident handle: trace loaded once; each step = rsim_rerun
    sizing = sizing_for(trace, cfg)
    for _ in range(6):
        h = _native.Handle(native_config(cfg, sizing, device=dev_index))
        h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
        try:
            h.rerun()
            break
        except _native.CapacityError:
            h.close()
            sizing = sizing.grown()
    for _ in range(max(args.warmup - 1, 0)):
        h.rerun()
    launches0 = h.launch_count()
    dev_ms, replay_ms, k1_ms = [], [], []
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            flush_l2(dev)
            dev_ms.append(h.rerun())
            tm = h.timings()
            replay_ms.append(tm[0])
            k1_ms.append(tm[1])
    launches = h.launch_count() - launches0
    ctr = h.counters()
    ns = h.decision_ns(0, R)
    lat = np.diff(ns[ns > 0]) / 1000.0
    chosen_dev, hit_dev = h.decisions(0, R)
    finish_dev = h.request_times(0, R)[2]
    whatif = measure_whatif(h, trace, cfg, args, name) if args.whatif else None
    h.close()

    # e2e through the public API run(records, config) (cluster.py:290-292): a new ClusterSim per
    # call (its device handle comes from the pool after the first), host arrays in, every
    # per-request result and the step log (record_steps=True, as the reference reports steps) out
    for _ in range(args.warmup):
        run(trace, cfg, device=dev_index)
    e2e_s = []
    for _ in range(args.steps):
        flush_l2(dev)
        t0 = time.perf_counter()
        rep = run(trace, cfg, device=dev_index)
        e2e_s.append(time.perf_counter() - t0)
    assert np.array_equal(rep.chosen, chosen_dev), "e2e and resident replays disagree"
    log_bytes = int(rep._step_log.nbytes) if rep._step_log is not None else 0
    release_pool()

    h2d = int(trace.arrival_us.nbytes + trace.in_tokens.nbytes + trace.out_tokens.nbytes +
              trace.request_id.nbytes + trace.blk_off.nbytes + trace.blocks.nbytes)
    d2h = R * (4 + 8 * 5) + log_bytes   # chosen, hit_tokens, first_sched, first_token, finish, route_bs + step log
    peaks, peak_src = measured_peaks()
    avg_replay_s = statistics.mean(replay_ms) / 1000.0
    achieved = ctr[0] / avg_replay_s / 1e9
    # K1 chain hashing: 16 B per prefix block (read hash, write key) + 8 B per
    # output-block key + 40 B of per-request metadata; timed by CUDA events inside each rerun
    nb = int(trace.blk_off[-1])
    nob = int(((trace.out_tokens + cfg.cache.block_size - 1) // cfg.cache.block_size).sum())
    k1_alg = 16 * nb + 8 * nob + 40 * R
    k1_s = statistics.mean(k1_ms) / 1000.0
    k1 = {"kernel": "k1_chain_keys", "prefix_blocks": nb, "output_keys": nob, "ms": k1_s * 1000.0,
          "keys_per_s": (nb + nob) / k1_s, "algorithmic_bytes": k1_alg,
          "roofline": {"bound": "hbm", "achieved": k1_alg / k1_s / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": k1_alg / k1_s / 1e9 / peaks["hbm_gbs"], "traffic": traffic_for(name, "k1_chain_keys"),
                       "l2": l2_for(name, "k1_chain_keys")}}
    out = {
        "R": R, "cfg": cfg, "trace": trace, "k1": k1,
        "value": R * len(dev_ms) / (sum(dev_ms) / 1000.0),
        "ms_per_step": statistics.mean(dev_ms),
        "e2e": R * len(e2e_s) / sum(e2e_s), "h2d": h2d, "d2h": d2h,
        "launches": launches, "clocks": clk.summary(), "whatif": whatif,
        "decisions_sha256_16": chosen_digest(chosen_dev),
        "lat_p50_us": float(np.percentile(lat, 50)) if lat.size else None,
        "lat_p99_us": float(np.percentile(lat, 99)) if lat.size else None,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": traffic_for(name),
                     "l2": l2_for(name, "replay_kernel"),
                     "kernel": "replay_kernel", "algorithmic_bytes_per_launch": int(ctr[0]),
                     "avg_launch_ms": avg_replay_s * 1000.0, "peak_source": f"{peak_src} hbm_gbs (burst copy)",
                     "engine_steps_per_launch": int(ctr[1])},
    }
    if with_cpu:
        n = reference_samples(trace, cfg, args.ref_budget_s)
        ref = time_reference(trace, cfg, n, repeats=3)      # best of 3
        cpu = host_cpu()
        if ref is not None:
            out["cpu_baseline"] = {"value": ref, "unit": "decisions/s", "cores": 1, "kind": "reference",
                                   "sample": f"first {n} of {R} requests, routesim.run from baseline/_ref (CPython, 1 thread), best of 3",
                                   "host_cpu": cpu}
    if args.parity:
        # the C oracle over the benched trace (or its first --parity-max requests): the timed CPU port
        # and the decision-by-decision parity check of this step's device replay
        sample = trace if R <= args.parity_max else trace.slice(args.parity_max)
        port, oref = time_port(sample, cfg)
        out["parity"] = parity_vs_oracle(oref, chosen_dev, hit_dev, finish_dev, R, _cutoff(trace, len(sample)))
        out["cpu_port"] = {"value": port, "unit": "decisions/s", "cores": 1, "kind": "port",
                           "sample": f"{'all' if len(sample) == R else 'first'} {len(sample)} of {R} requests, "
                                     "oracle/rsim_oracle.c (1 thread)", "host_cpu": host_cpu()}
        if "cpu_baseline" not in out and with_cpu:
            out["cpu_baseline"] = dict(out["cpu_port"])
    return out


def measure_route_api(name, n_calls, dev_index, with_ref: bool):
    """The online router use case (BASELINE.md section 2 route p50/p99): ``ClusterSim.route(record,
    now_us)`` called once per request in arrival order, each call timed with perf_counter_ns around
    the public API (host record in, RoutingDecision with every instance's score out); the reference's
    ``ClusterSim.route`` on the same records beside it, and the two decision sequences compared."""
    from paper_2603_15202_b200.cluster import ClusterSim
    trace, cfg = build_workload(name)
    recs = trace.slice(min(n_calls, len(trace))).records()
    arr = [int(x) for x in trace.arrival_us[:len(recs)]]
    warm = ClusterSim(cfg, device=dev_index)
    for r, t in zip(recs[:32], arr[:32]):
        warm.route(r, t)
    warm.close()
    sim = ClusterSim(cfg, device=dev_index)
    ns, chosen = [], []
    for r, t in zip(recs, arr):
        t0 = time.perf_counter_ns()
        d = sim.route(r, t)
        ns.append(time.perf_counter_ns() - t0)
        chosen.append(d.chosen)
    sim.close()
    us = np.asarray(ns) / 1000.0
    # the same calls straight through the C ABI (rsim_route_request): the boundary's own cost
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.cluster import native_config, sizing_for
    h = _native.Handle(native_config(cfg, sizing_for(trace.slice(len(recs)), cfg), device=dev_index))
    blk = [np.asarray(r.prefix_blocks, np.uint64) for r in recs]
    cns = []
    for r, b, t in zip(recs, blk, arr):
        t0 = time.perf_counter_ns()
        h.route_request(t, r.input_tokens, r.output_tokens, r.request_id, b)
        cns.append(time.perf_counter_ns() - t0)
    h.close()
    cus = np.asarray(cns) / 1000.0
    out = {"instances": cfg.n_instances, "calls": len(recs), "workload": name,
           "c_abi": {"p50_us": float(np.percentile(cus, 50)), "p99_us": float(np.percentile(cus, 99)),
                     "entry": "rsim_route_request"},
           "ours": {"p50_us": float(np.percentile(us, 50)), "p99_us": float(np.percentile(us, 99)),
                    "mean_us": float(us.mean()), "calls_per_s": len(us) / (us.sum() / 1e6)},
           "timed": "perf_counter_ns around each ClusterSim.route(record, now_us) call (no engine steps between "
                    "calls, as in the reference's route()); ours: host record -> RoutingDecision incl. scores"}
    if with_ref and import_reference() is not None:
        routesim, rrecs, rcfg = ref_records_and_config(trace.slice(len(recs)), cfg)
        from routesim.cluster import ClusterSim as RefSim
        ref = RefSim(rcfg)
        rns, rchosen = [], []
        for r, t in zip(rrecs, arr):
            t0 = time.perf_counter_ns()
            d = ref.route(r, t)
            rns.append(time.perf_counter_ns() - t0)
            rchosen.append(d.chosen)
        rus = np.asarray(rns) / 1000.0
        out["reference"] = {"p50_us": float(np.percentile(rus, 50)), "p99_us": float(np.percentile(rus, 99)),
                            "mean_us": float(rus.mean()), "calls_per_s": len(rus) / (rus.sum() / 1e6),
                            "impl": "routesim ClusterSim.route from baseline/_ref (CPython, 1 thread)"}
        out["parity"] = {"vs": "reference ClusterSim.route", "calls": len(recs),
                         "mismatches": int(sum(a != b for a, b in zip(chosen, rchosen)))}
        out["p50_speedup"] = out["reference"]["p50_us"] / out["ours"]["p50_us"]
    return out


def measure_whatif(h, trace, cfg, args, name):
    """SURVEY 8d tertiary: the batched what-if probe (M requests x all instances against the
    replay's final KV$ state, no commits) -- the bandwidth-bound form of the probe.
    Algorithmic bytes: 8 B per chain key of each request (read once) + 8 B per
    reference dict lookup, min(h+1, B) per (request, instance)."""
    M = min(len(trace), args.whatif)
    hits = h.probe_batch(0, M)                       # warm-up + the hit matrix
    ms = []
    for _ in range(3):
        h.probe_batch(0, M)
        ms.append(h.timings()[0])
    B = np.diff(trace.blk_off[:M + 1]).astype(np.int64)
    look = np.minimum(hits.astype(np.int64) + 1, B[:, None])
    alg = int(8 * B.sum() + 8 * look.sum())
    best = min(ms) / 1000.0
    peaks, _ = measured_peaks()
    gbs = alg / best / 1e9
    kern = "probe_scan_kernel"
    return {"requests": M, "instances": int(hits.shape[1]), "pairs": int(M * hits.shape[1]),
            "ms": min(ms), "pairs_per_s": M * hits.shape[1] / best, "algorithmic_bytes": alg,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"], "kernel": kern, "traffic": traffic_for(name, kern),
                         "l2": l2_for(name, kern)}}


def traffic_for(name, kernel="replay_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of ``kernel`` on this workload, from
    the committed ncu capture (profiles/kernel_traffic.json, tools/profile_r2.sh +
    tools/update_traffic.py); None if not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_traffic.json")) as fh:
            t = json.load(fh).get(name, {}).get(kernel)
        return None if t is None else int(t["dram_bytes"])
    except (OSError, ValueError, KeyError):
        return None


def l2_for(name, kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_traffic.json")) as fh:
            t = json.load(fh).get(name, {}).get(kernel)
        return None if t is None else {"l2_sector_bytes": 32 * int(t["l2_sectors"]), "l2_hit_pct": t["l2_hit_pct"]}
    except (OSError, ValueError, KeyError):
        return None


def peer_evidence(rank, world, dev_index, router, backend):
    """Per-rank device identity and peer-open evidence (the data plane is not NCCL, so the
    driver's comm_nranks_ok says nothing about it)."""
    import torch
    p = torch.cuda.get_device_properties(dev_index)
    ndev = torch.cuda.device_count()
    peers = {}
    for r in range(world):
        d = r % ndev
        if r != rank:
            peers[str(r)] = {"device": d, "same_device": d == dev_index,
                             "can_access_peer": bool(d == dev_index or torch.cuda.can_device_access_peer(dev_index, d))}
    return {"rank": rank, "device": dev_index, "name": p.name, "pci_bus_id": getattr(p, "pci_bus_id", None),
            "uuid": str(getattr(p, "uuid", "")), "shard": list(router.h.shard_bounds()),
            "ipc_mailboxes_opened": router.peers_opened, "plumbing_backend": backend, "peers": peers}


def measure_sharded(name, args, dev_index, rank, world, backend):
    """Instances of one cluster sharded over `world` GPUs (one process each); per decision every
    rank publishes its (min score, tie count) partial into every peer's mailbox over NVLink
    (device-initiated, distributed.py). Strong scaling: the total work is the one trace."""
    import torch
    import torch.distributed as dist
    from paper_2603_15202_b200.distributed import ShardedRouter

    trace, cfg = build_workload(name)
    if args.requests and args.requests < len(trace):
        trace = trace.slice(args.requests)
    R = len(trace)
    dev = torch.device("cuda", dev_index)
    router = ShardedRouter(cfg, trace, rank=rank, world=world, device=dev_index)
    for _ in range(args.warmup):
        router.rerun()
    launches0 = router.h.launch_count()
    dev_ms, replay_ms, k1_ms = [], [], []
    with ClockSampler(dev_index) as clk:
        for _ in range(args.steps):
            flush_l2(dev)
            dist.barrier()
            dev_ms.append(router.rerun())
            tm = router.h.timings()
            replay_ms.append(tm[0])
            k1_ms.append(tm[1])
    launches = router.h.launch_count() - launches0
    ctr = router.h.counters()
    ns = router.h.decision_ns(0, R)                  # this rank's clock, stamped at every decide
    lat = np.diff(ns[ns > 0]) / 1000.0
    ch_local, ht_local = router.local_decisions()
    fin_local = router.h.request_times(0, R)[2]
    evidence = peer_evidence(rank, world, dev_index, router, backend)
    e2e_s = []
    for _ in range(args.steps):
        flush_l2(dev)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chosen, hit_tokens = router.run_trace(trace)
        e2e_s.append(time.perf_counter() - t0)
    router.close()
    # merge this rank's owned decisions with its peers' (each decision is committed by exactly one rank)
    fin = merge_over_ranks(fin_local, backend, dev)
    assert np.array_equal(merge_over_ranks(ch_local.astype(np.int64), backend, dev).astype(np.int32), chosen), \
        "resident and e2e sharded replays disagree"
    h2d = int(trace.arrival_us.nbytes + trace.in_tokens.nbytes + trace.out_tokens.nbytes +
              trace.request_id.nbytes + trace.blk_off.nbytes + trace.blocks.nbytes)
    peaks, peak_src = measured_peaks()
    avg_replay_s = statistics.mean(replay_ms) / 1000.0
    achieved = ctr[0] / avg_replay_s / 1e9 if avg_replay_s else 0.0
    nb = int(trace.blk_off[-1])
    nob = int(((trace.out_tokens + cfg.cache.block_size - 1) // cfg.cache.block_size).sum())
    k1_alg = 16 * nb + 8 * nob + 40 * R
    k1_s = statistics.mean(k1_ms) / 1000.0
    k1 = {"kernel": "k1_chain_keys", "prefix_blocks": nb, "output_keys": nob, "ms": k1_s * 1000.0,
          "keys_per_s": (nb + nob) / k1_s, "algorithmic_bytes": k1_alg, "scope": "replicated on every rank",
          "roofline": {"bound": "hbm", "achieved": k1_alg / k1_s / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": k1_alg / k1_s / 1e9 / peaks["hbm_gbs"], "traffic": traffic_for(name, "k1_chain_keys"),
                       "l2": l2_for(name, "k1_chain_keys")}}
    out = {"R": R, "cfg": cfg, "trace": trace, "k1": k1, "ms_per_step": statistics.mean(dev_ms),
           "e2e_s": statistics.mean(e2e_s), "h2d": h2d, "d2h": R * 12, "launches": launches,
           "clocks": clk.summary(), "chosen": chosen, "hit_tokens": hit_tokens, "finish_us": fin,
           "evidence": evidence,
           "lat_p50_us": float(np.percentile(lat, 50)) if lat.size else None,
           "lat_p99_us": float(np.percentile(lat, 99)) if lat.size else None,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": achieved / peaks["hbm_gbs"], "traffic": None, "kernel": "replay_kernel",
                        "algorithmic_bytes_per_launch": int(ctr[0]), "avg_launch_ms": avg_replay_s * 1000.0,
                        "peak_source": f"{peak_src} hbm_gbs (burst copy)", "scope": f"rank {rank} shard"}}
    return out


def merge_over_ranks(a, backend, dev):
    """Element-wise max over ranks (non-owned entries are -1)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64))
    t = t.to(dev) if backend == "nccl" else t
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def relaunch_distributed(n):
    """``bench.py --gpus N`` outside torchrun: re-exec under torch.distributed.run with N ranks."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def default_workload(world):
    """api64 (BASELINE configs[1], where the metric is quoted) on one GPU; the sharded configs[3]
    cluster (4096 instances over the N GPUs) for N > 1."""
    return "api64" if world == 1 else "large4096"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: api64 on 1 GPU, large4096 sharded over N > 1")
    ap.add_argument("--requests", type=int, default=0, help="sharded runs: replay only the first R requests (0: all)")
    ap.add_argument("--extra", default="chat1024,agent256,adv64", help="comma list of extra workloads reported beside the headline")
    ap.add_argument("--ref-budget-s", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", dest="parity", action="store_false",
                    help="skip the decision-by-decision check of the device replay against the C oracle")
    ap.add_argument("--parity-max", type=int, default=0,
                    help="oracle-checked prefix length (decision k depends only on records[:k+1]); "
                         "default 120k on 1 GPU (every request of api64 / chat1024 / agent256), 50k sharded")
    ap.add_argument("--route-api", default="api64:2000,chat1024:500",
                    help="online route() API latency, workload:calls list ('' to skip)")
    ap.add_argument("--whatif", type=int, default=20000,
                    help="requests of the batched what-if probe measured after the replay (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    if world > 1 and args.gpus not in (1, world):
        raise SystemExit(f"--gpus {args.gpus} does not match WORLD_SIZE={world}")
    if args.workload is None:
        args.workload = default_workload(world)
    if args.parity_max <= 0:
        args.parity_max = 120_000 if world == 1 else 50_000
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    ndev = torch.cuda.device_count()
    dev_index = local % max(ndev, 1)                 # ranks share a GPU only when fewer GPUs than ranks
    torch.cuda.set_device(dev_index)
    from paper_2603_15202_b200 import workloads as W
    W.use_device_generator(dev_index)                # synthetic traces built on the GPU (bit-identical)
    pg, backend = None, None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if ndev >= world else "gloo"   # NCCL cannot put two ranks on one device
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
        pg = dist
        pg.barrier()
    torch.cuda.synchronize()
    if world > 1:
        res = measure_sharded(args.workload, args, dev_index, rank, world, backend)
    else:
        res = measure_workload(args.workload, args, dev_index, with_cpu=not args.no_cpu, rank=rank)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
        t = torch.tensor([res["ms_per_step"], res["e2e_s"]], dtype=torch.float64)
        t = t.cuda() if backend == "nccl" else t
        pg.all_reduce(t, op=pg.ReduceOp.MAX)          # max over ranks
        res["ms_per_step"], res["e2e_s"] = float(t[0].item()), float(t[1].item())
        res["e2e"] = res["R"] / res["e2e_s"]
        ev = [None] * world
        pg.all_gather_object(ev, res["evidence"])
        res["evidence"] = ev
        if rank == 0 and args.parity:
            trace, cfg = res["trace"], res["cfg"]
            sample = trace if res["R"] <= args.parity_max else trace.slice(args.parity_max)
            port, oref = time_port(sample, cfg)
            res["parity"] = parity_vs_oracle(oref, res["chosen"], res["hit_tokens"], res["finish_us"], res["R"],
                                             _cutoff(trace, len(sample)))
            res["cpu_port"] = {"value": port, "unit": "decisions/s", "cores": 1, "kind": "port",
                               "sample": f"first {len(sample)} of {res['R']} requests, oracle/rsim_oracle.c (1 thread)",
                               "host_cpu": host_cpu()}
        res["decisions_sha256_16"] = chosen_digest(res["chosen"])
    extras = {}
    route_api = None
    if world == 1 and args.route_api:
        route_api = [measure_route_api(spec.split(":")[0], int(spec.split(":")[1]), dev_index, with_ref=not args.no_cpu)
                     for spec in args.route_api.split(",") if spec]
    if world == 1:
        for name in [x for x in args.extra.split(",") if x and x != args.workload]:
            e = measure_workload(name, args, dev_index, with_cpu=not args.no_cpu, rank=rank)
            extras[name] = {"value": e["value"], "e2e": e["e2e"], "ms_per_step": e["ms_per_step"],
                            "n_instances": e["cfg"].n_instances, "requests": e["R"],
                            "decision_latency_us": {"p50": e["lat_p50_us"], "p99": e["lat_p99_us"]},
                            "parity": e.get("parity"), "decisions_sha256_16": e.get("decisions_sha256_16"),
                            "roofline": e["roofline"], "whatif_probe": e.get("whatif"), "k1_chain_keys": e["k1"],
                            "cpu_baseline": e.get("cpu_baseline"),
                            "cpu_port": e.get("cpu_port"),
                            "e2e_vs_cpu_baseline": (e["e2e"] / e["cpu_baseline"]["value"]) if e.get("cpu_baseline") else None,
                            "description": WORKLOADS[name][1]}
    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    R = res["R"]
    value = R / (res["ms_per_step"] / 1000.0)          # decisions of the one (sharded) cluster per second
    line = {
        "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": args.workload, "description": WORKLOADS[args.workload][1],
                   "n_instances": res["cfg"].n_instances, "requests": R, "block_size": res["cfg"].cache.block_size,
                   "capacity_blocks": res["cfg"].cache.capacity_blocks, "policy": res["cfg"].policy.kind,
                   "parallelism": (f"instances sharded over {world} ranks ({backend} plumbing), per-decision "
                                   "device-initiated mailbox exchange over peer memory") if world > 1 else "single-gpu",
                   "l2": "512 MB flush between timed steps; trace + tables exceed L2"},
        "decision_latency_us": {"p50": res["lat_p50_us"], "p99": res["lat_p99_us"],
                                "source": "%globaltimer at each commit (rank 0's decide for N > 1), consecutive differences"},
        "parity": res.get("parity"),
        "decisions_sha256_16": res.get("decisions_sha256_16"),
        "roofline": res["roofline"],
        "e2e": {"value": res["e2e"], "unit": "decisions/s", "h2d_bytes_per_step": res["h2d"],
                "d2h_bytes_per_step": res["d2h"]},
        "gpu_launches": res["launches"],
        "whatif_probe": res.get("whatif"), "k1_chain_keys": res["k1"],
        "route_api": route_api,
        "clocks": res["clocks"],
    }
    if world > 1:
        line["ranks"] = res["evidence"]
    if "cpu_baseline" in res:
        line["cpu_baseline"] = res["cpu_baseline"]
        line["e2e_vs_cpu_baseline"] = res["e2e"] / res["cpu_baseline"]["value"]
    if "cpu_port" in res:
        line["cpu_port"] = res["cpu_port"]
    if extras:
        line["extra_workloads"] = extras
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()

if __name__ == "__main__":
    main()
