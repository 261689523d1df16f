"""Time (or profile under ncu) one resident replay of a workload slice.

    python tools/profile_replay.py api64 20000 [ctas warps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_15202_b200 import _native  # noqa: E402
from paper_2603_15202_b200.cluster import native_config, sizing_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "api64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
shapes = [(int(sys.argv[3]), int(sys.argv[4]))] if len(sys.argv) > 4 else [(0, 0)]
world = int(sys.argv[5]) if len(sys.argv) > 5 else 1
if len(sys.argv) > 3 and sys.argv[3] == "sweep":
    shapes = [(c, w) for c in (1, 2, 4, 8, 16) for w in (4, 8, 16)]
burst = name.endswith("-burst")            # all arrivals at t=0: no engine steps, pure route cost
trace, cfg = bench.build_workload(name.replace("-burst", ""))
trace = trace.slice(min(n, len(trace)))
if burst:
    import numpy as np
    from paper_2603_15202_b200.trace import PackedTrace
    trace = PackedTrace(trace.request_id, np.zeros_like(trace.arrival_s), trace.in_tokens, trace.out_tokens,
                        trace.class_key, trace.blk_off, trace.blocks)
if world > 1:
    from paper_2603_15202_b200.distributed import run_sharded_local
    for c, w in shapes:
        r = run_sharded_local(trace, cfg, world, ctas=c, warps_per_cta=w, repeats=3)
        best = min(r["device_ms"])
        print(f"{name} R={len(trace)} world={world} ctas={c} warps={w}: total {best:.2f} ms "
              f"({1000 * best / len(trace):.2f} us/decision)", flush=True)
    sys.exit(0)
def critpath(h, n):
    """Per decision: the warp whose partial came last (largest release->publish latency) and why."""
    import numpy as np
    h.phase_records(n)
    h.rerun()
    rec = h.read_phase_records(n).astype(np.float64)          # [n, warps, 8]
    lat = rec[:, :, 0]
    mx = lat.argmax(axis=1)
    top = rec[np.arange(n), mx]                                # record of the slowest warp
    med = np.median(lat, axis=1)
    print(f"   critical warp (cycles): latency {16 * top[:, 0].mean():.0f} (median warp {16 * med.mean():.0f})"
          f"  stage-wait {16 * top[:, 3].mean():.0f}  drain {16 * top[:, 1].mean():.0f}  probe+score {16 * top[:, 2].mean():.0f}"
          f"  rest {16 * (top[:, 0] - top[:, 1] - top[:, 2] - top[:, 3]).mean():.0f}", flush=True)
    print(f"   critical warp: steps {top[:, 4].mean():.2f}/decision, finisher batches {top[:, 5].mean():.2f}, "
          f"parked batches {top[:, 7].mean():.2f}, previous owner {top[:, 6].mean():.2f}; all warps: steps "
          f"{rec[:, :, 4].sum(1).mean():.2f}, finisher batches {rec[:, :, 5].sum(1).mean():.2f}, parked "
          f"{rec[:, :, 7].sum(1).mean():.2f}", flush=True)
    for own in (0, 1):
        m = top[:, 6] == own
        if m.any():
            print(f"     critical warp {'is' if own else 'is not'} the previous owner: {m.mean():.2f} of decisions, latency "
                  f"{16 * top[m, 0].mean():.0f}, stage-wait {16 * top[m, 3].mean():.0f}, drain {16 * top[m, 1].mean():.0f}, "
                  f"probe {16 * top[m, 2].mean():.0f}, steps {top[m, 4].mean():.2f}, parked {top[m, 7].mean():.2f}", flush=True)
    for lo, hi in ((0, 1), (1, 2), (2, 99)):
        m = (top[:, 5] >= lo) & (top[:, 5] < hi)
        if m.any():
            print(f"     critical warp with {lo}{'+' if hi > 2 else ''} finisher batches: {m.mean():.2f} of decisions, latency "
                  f"{16 * top[m, 0].mean():.0f}, drain {16 * top[m, 1].mean():.0f}, probe {16 * top[m, 2].mean():.0f}, "
                  f"steps {top[m, 4].mean():.2f}", flush=True)
    tl = h.read_phase_times(n, rec.shape[1]).astype(np.float64)   # ns
    W = rec.shape[1]
    pub = tl[:, :W].max(axis=1)
    land, decided, rel = tl[:, W], tl[:, W + 1], tl[:, W + 2]
    ok = (land > 0) & (decided > 0) & (rel > 0)
    ok[1:] &= rel[:-1] > 0
    idx = np.nonzero(ok[1:])[0] + 1
    if idx.size:
        f = lambda x: float(np.median(x))
        print(f"   timeline (median ns per decision): period {f(rel[idx] - rel[idx - 1]):.0f} = release->last publish "
              f"{f(pub[idx] - rel[idx - 1]):.0f} + exchange {f(land[idx] - pub[idx]):.0f} + decide {f(decided[idx] - land[idx]):.0f}"
              f" + release {f(rel[idx] - decided[idx]):.0f}", flush=True)
    h.phase_records(0)


for c, w in shapes:
    if c and c > cfg.n_instances:
        continue
    try:
        h = _native.Handle(native_config(cfg, sizing_for(trace, cfg), ctas=c, warps_per_cta=w, record_steps=bool(os.environ.get("RSIM_LOG")), step_log_capacity=(8 * len(trace) + int(trace.out_tokens.sum()) // 2) if os.environ.get("RSIM_LOG") else 0))
    except ValueError as exc:
        print(f"{name} ctas={c} warps={w}: skipped ({exc})")
        continue
    h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)
    if cfg.detector is not None:
        from paper_2603_15202_b200.cluster import detector_classes
        tid, off, ln, key = detector_classes(trace, cfg.detector.class_key_blocks)
        h.load_detector(tid, off, ln, key, 1 << 16)
    h.rerun()
    best = min(h.rerun() for _ in range(3))
    if os.environ.get("RSIM_CRIT"):
        critpath(h, len(trace))
    rep, k1, dr = h.timings()
    print(f"{name} R={len(trace)} ctas={c} warps={w}: total {best:.2f} ms  replay {rep:.2f} ms "
          f"({1000 * rep / len(trace):.2f} us/decision)  k1 {k1:.3f} ms  drain {dr:.2f} ms", flush=True)
    ctr = h.counters()
    names = ["stage", "drain", "probe", "pub+spec", "xwait", "decide", "barrier", "commit"]
    cyc = ctr[8:16].astype(float) / len(trace)
    print("   cycles/decision (CTA0 warp0): " + "  ".join(f"{n}={c:.0f}" for n, c in zip(names, cyc))
          + f"  sum={cyc.sum():.0f}", flush=True)
    if ctr[1]:
        print(f"   engine: {ctr[1] / len(trace):.2f} steps/decision, {ctr[2] / max(ctr[1], 1):.0f} cycles/step, "
              f"{ctr[6]} finisher batches at {ctr[3] / max(ctr[6], 1):.0f} cycles each", flush=True)
    sc = h.step_cycles()
    if sc.any() and ctr[1]:
        names = ["setup", "plan", "cost", "apply", "pops", "decode", "finish", "joins+tail"]
        print("   step sections (cycles/step): " + "  ".join(f"{n}={c / ctr[1]:.0f}" for n, c in zip(names, sc[:8])), flush=True)
        if sc[14] or sc[15]:
            print(f"   warp 0 post-publish: advance non-candidates {sc[14] / len(trace):.0f} cyc/decision, "
                  f"probe-ahead {sc[15] / len(trace):.0f} cyc/decision", flush=True)
        if sc[16] or sc[17]:
            print(f"   warp 0 probe-ahead sections: setup {sc[16] / len(trace):.0f}  issue {sc[17] / len(trace):.0f}  "
                  f"evaluate {sc[18] / len(trace):.0f} cyc/decision", flush=True)
        if sc[19] or sc[20]:
            print(f"   decide sections (CTA 0 control warp, cyc/decision): load+min {sc[19] / len(trace):.0f}  "
                  f"ties+index {sc[20] / len(trace):.0f}  owner {sc[21] / len(trace):.0f}", flush=True)
        if sc[22] or sc[23]:
            print(f"   detector (CTA 0 control warp, cyc/decision): listed-holder wait {sc[22] / len(trace):.0f}  "
                  f"observe {sc[23] / len(trace):.0f}  prepare {sc[24] / len(trace):.0f}; decisions with a list "
                  f"{sc[25] / len(trace):.2f}", flush=True)
        if sc[26] or sc[27]:
            print(f"   inline finishes (finish_one): insert {sc[26] / max(ctr[6], 1):.0f} cyc/batch, evict {sc[27] / max(ctr[6], 1):.0f} "
                  f"cyc/batch; evict walk: {sc[31]} groups, {sc[28]} batches, {sc[29]} victims, delete {sc[30] / max(sc[29], 1):.0f} cyc/victim",
                  flush=True)
        kinds = ["finishing", "other full", "pure decode"]
        print("   step kinds: " + "  ".join(f"{kinds[i]} {sc[8 + 2 * i]} x {sc[9 + 2 * i] / max(sc[8 + 2 * i], 1):.0f} cyc"
                                          for i in range(3)), flush=True)
    h.close()
