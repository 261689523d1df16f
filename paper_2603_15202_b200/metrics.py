"""Run analytics over the device Collector columns: ``summarize`` / ``export`` with the
reference's file set and byte-stable contents (reference metrics.py:1-14, 162-497).

The reference walks Python objects (``report.requests``, ``report.steps``,
``report.bs_series``); here every statistic is computed from the columns the replay
kernel wrote (per-request times, the step log, the per-route batch sizes) without
materialising them. Floating-point results are bit-identical to the reference's:
element-wise operations are the same IEEE operations on the same (exactly
representable) integers, sums that the reference takes with Python's ``sum`` (compensated
since CPython 3.12) are taken with ``sum`` here too, accumulations the reference does in
a loop (+=, per window and instance) keep their order (``np.add.at`` is unbuffered), and
standard deviations go through the same ``statistics.pstdev``.
"""

from __future__ import annotations

import csv
import json
import math
import statistics
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .report import RunReport, percentile

__all__ = ["summarize", "export", "percentile", "hit_timeline", "imbalance_profile", "prefill_imbalance_std",
           "mean_bs_by_instance", "bs_spread", "WindowProfile", "REQUEST_COLUMNS"]

REQUEST_COLUMNS = ("request_id", "arrival_s", "chosen_instance", "class_key", "input_tokens", "output_tokens",
                   "hit_ratio", "ttft_ms", "tpot_ms", "queue_delay_ms", "first_token_s", "finish_s")


@dataclass(frozen=True)
class WindowProfile:
    window_start_s: float
    prefill_s: dict
    mean_bs: dict
    hit_ratio: float | None


# ---------------------------------------------------------------- columns
class _Cols:
    """Per-request columns (request order) of a RunReport."""

    def __init__(self, rep: RunReport):
        tr, c = rep._trace, rep.columns
        n = 0 if tr is None else len(tr)
        z = np.zeros(0, np.int64)
        self.n = n
        self.rid = tr.request_id if n else z.astype(np.uint64)
        self.cls = tr.class_key if n else z.astype(np.uint64)
        self.arr = tr.arrival_us if n else z
        self.inp = tr.in_tokens if n else z
        self.out = tr.out_tokens if n else z
        self.chosen = c["chosen"] if n else z
        self.hit = c["hit_tokens"] if n else z
        self.fs = c["first_sched_us"] if n else z
        self.ft = c["first_token_us"] if n else z
        self.fin = c["finish_us"] if n else z

    def ttft_us(self):                                       # RequestMetrics.ttft_us (metrics.py:45-47)
        m = self.ft >= 0
        return m, self.ft - self.arr

    def tpot_us(self):                                       # RequestMetrics.tpot_us (metrics.py:50-56)
        m = (self.fin >= 0) & (self.ft >= 0) & (self.out >= 2)
        num = (self.fin - self.ft).astype(np.float64)
        den = np.where(m, self.out - 1, 1).astype(np.float64)
        return m, num / den

    def hit_ratio(self):
        return self.hit.astype(np.float64) / self.inp.astype(np.float64)


def _cols(rep: RunReport) -> _Cols:
    c = getattr(rep, "_metric_cols", None)
    if c is None:
        c = _Cols(rep)
        rep._metric_cols = c
    return c


def _bs_events(rep: RunReport):
    """bs_series as flat event arrays (inst, t, bs) in the order the reference appends them:
    routes (arrival, bs after enqueue) and step launches (start, bs), sorted like report.bs_series."""
    c = _cols(rep)
    log = rep._sorted_log()
    rmask = c.chosen >= 0
    k = np.nonzero(rmask)[0]
    rb = rep.columns.get("route_bs") if c.n else None
    t = np.concatenate([c.arr[k], log[:, 1]])
    kind = np.concatenate([np.zeros(k.size, np.int64), np.ones(len(log), np.int64)])
    idx = np.concatenate([k.astype(np.int64), log[:, 5]])
    inst = np.concatenate([c.chosen[k].astype(np.int64), log[:, 0]])
    bs = np.concatenate([(rb[k] if rb is not None else np.zeros(k.size, np.int64)).astype(np.int64), log[:, 4]])
    order = np.lexsort((bs, inst, idx, kind, t))           # ev.sort() on (t, kind, i, inst, bs)
    return inst[order], t[order], bs[order]


def _window_count(end_us: int, window_us: int) -> int:
    return max(1, -(-end_us // window_us)) if end_us > 0 else 0


# ---------------------------------------------------------------- statistics
def mean_bs_by_instance(rep: RunReport) -> dict:
    """Time-weighted mean batch size per instance (reference metrics.py:173-188)."""
    horizon = rep.end_us
    inst, t, bs = _bs_events(rep)
    out = {}
    for i in range(rep.n_instances):
        if horizon <= 0:
            out[i] = 0.0
            continue
        m = inst == i
        ti, bi = t[m], bs[m]
        prev_t = np.concatenate([[0], ti])
        prev_b = np.concatenate([[0], bi])
        nxt = np.concatenate([ti, [horizon]])
        area = int((prev_b * (nxt - prev_t)).sum())          # exact integer area
        out[i] = area / horizon
    return out


def bs_spread(rep: RunReport):
    means = list(mean_bs_by_instance(rep).values())
    if not means:
        return None
    hi, lo = max(means), min(means)
    if hi == 0.0:
        return 1.0
    if lo == 0.0:
        return math.inf
    return hi / lo


def hit_timeline(rep: RunReport, window_s: float = 10.0, request_weighted: bool = False):
    """Per-window (start_s, hit_ratio, hit_tokens, input_tokens) (reference metrics.py:298-323)."""
    window_us = int(window_s * 1e6)
    n_win = _window_count(rep.end_us, window_us)
    if n_win == 0:
        return []
    c = _cols(rep)
    w = np.minimum(c.arr // window_us, n_win - 1)
    hit_tok = np.zeros(n_win, np.int64)
    in_tok = np.zeros(n_win, np.int64)
    np.add.at(hit_tok, w, c.hit)
    np.add.at(in_tok, w, c.inp)
    hr = c.hit_ratio() if request_weighted else None
    rows = []
    for j in range(n_win):
        if request_weighted:
            sel = hr[w == j].tolist()
            ratio = sum(sel) / len(sel) if sel else None
        else:
            ratio = int(hit_tok[j]) / int(in_tok[j]) if in_tok[j] else None
        rows.append((j * window_us / 1e6, ratio, int(hit_tok[j]), int(in_tok[j])))
    return rows


def imbalance_profile(rep: RunReport, window_s: float = 10.0):
    """Windowed prefill seconds and mean bs per instance + the two instances with the
    largest stddev of windowed prefill time (reference metrics.py:216-283)."""
    window_us = int(window_s * 1e6)
    n_win = _window_count(rep.end_us, window_us)
    N = rep.n_instances
    prefill = np.zeros(n_win * N, np.float64)
    log = rep._sorted_log()
    if n_win and len(log):
        inst, s, e, pre = log[:, 0], log[:, 1], log[:, 2], log[:, 3]
        keep = (e > s) & (pre != 0)
        inst, s, e, pre = inst[keep], s[keep], e[keep], pre[keep]
        # split every step at window boundaries, pieces in step order (the reference's loop order)
        w0 = s // window_us
        nw = (e - 1) // window_us - w0 + 1
        rep_idx = np.repeat(np.arange(len(s)), nw)
        wi = w0[rep_idx] + (np.arange(rep_idx.size) - np.repeat(np.cumsum(nw) - nw, nw))
        lo = np.maximum(s[rep_idx], wi * window_us)
        hi = np.minimum(e[rep_idx], (wi + 1) * window_us)
        val = (pre[rep_idx] * (hi - lo)).astype(np.float64) / (e - s)[rep_idx].astype(np.float64) / 1e6
        ok = wi < n_win
        np.add.at(prefill, wi[ok] * N + inst[rep_idx][ok], val[ok])
    prefill = prefill.reshape(n_win, N) if n_win else prefill.reshape(0, N)

    mean_bs = np.zeros((n_win, N), np.int64)
    if n_win:
        ev_inst, ev_t, ev_bs = _bs_events(rep)
        for i in range(N):
            m = ev_inst == i
            ts = np.concatenate([[0], ev_t[m], [rep.end_us]])
            bs = np.concatenate([[0], ev_bs[m], [0]])
            a, b, v = ts[:-1], ts[1:], bs[:-1]
            seg = (b > a) & (v != 0)
            for pt, t, pb in zip(a[seg].tolist(), b[seg].tolist(), v[seg].tolist()):
                w = pt // window_us
                while w * window_us < t:
                    l, h = max(pt, w * window_us), min(t, (w + 1) * window_us)
                    if w < n_win:
                        mean_bs[w, i] += pb * (h - l)
                    w += 1

    hits = {row[0]: row[1] for row in hit_timeline(rep, window_s)}
    profiles = []
    for w in range(n_win):
        start_us = w * window_us
        covered = min((w + 1) * window_us, rep.end_us) - start_us
        pw = prefill[w].tolist()
        mb = mean_bs[w].tolist()
        profiles.append(WindowProfile(start_us / 1e6, {i: pw[i] for i in range(N)},
                                      {i: (mb[i] / covered if covered > 0 else 0.0) for i in range(N)},
                                      hits.get(start_us / 1e6)))
    if N < 2 or n_win == 0:
        return profiles, (0, 0)
    cols = prefill.T.tolist()
    stds = [statistics.pstdev(cols[i]) if n_win > 1 else 0.0 for i in range(N)]
    ranked = sorted(range(N), key=lambda i: (-stds[i], i))
    return profiles, (ranked[0], ranked[1])


def prefill_imbalance_std(rep: RunReport, window_s: float = 10.0):
    profiles, _ = imbalance_profile(rep, window_s)
    if not profiles or rep.n_instances < 2:
        return None
    per = [statistics.pstdev([p.prefill_s[i] for i in range(rep.n_instances)]) for p in profiles]
    return sum(per) / len(per)


def _stats(series: list):
    if not series:
        return {"mean": None, "p50": None, "p95": None, "p99": None}
    xs = sorted(series)

    def pct(p):
        return xs[max(math.ceil(p / 100.0 * len(xs)), 1) - 1]
    return {"mean": sum(series) / len(series), "p50": pct(50), "p95": pct(95), "p99": pct(99)}


def summarize(rep: RunReport, request_weighted_hits: bool = False) -> dict:
    """summary.json contents (reference metrics.py:342-380)."""
    c = _cols(rep)
    m, tt = c.ttft_us()
    ttft = (tt[m].astype(np.float64) / 1000.0).tolist()
    m2, tp = c.tpot_us()
    tpot = (tp[m2] / 1000.0).tolist()
    t, o = _stats(ttft), _stats(tpot)
    spread = bs_spread(rep)
    if c.n == 0:
        hit = None
    elif request_weighted_hits:
        hit = sum(c.hit_ratio().tolist()) / c.n
    else:
        hit = int(c.hit.sum()) / int(c.inp.sum())
    return {
        "policy": rep.policy_kind, "seed": rep.seed, "n_instances": rep.n_instances, "routed": rep.routed,
        "finished": rep.finished, "queued_at_last_arrival": rep.queued_at_last_arrival,
        "arrivals_hash": rep.arrivals_hash, "sim_end_s": rep.end_us / 1e6, "hit_ratio": hit,
        "ttft_count": len(ttft), "mean_ttft_ms": t["mean"], "p50_ttft_ms": t["p50"], "p95_ttft_ms": t["p95"],
        "p99_ttft_ms": t["p99"],
        "tpot_count": len(tpot), "mean_tpot_ms": o["mean"], "p50_tpot_ms": o["p50"], "p95_tpot_ms": o["p95"],
        "p99_tpot_ms": o["p99"],
        "mean_bs_spread": None if spread is None or math.isinf(spread) else spread,
        "prefill_imbalance_std_s": prefill_imbalance_std(rep),
    }


# ---------------------------------------------------------------- export
def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _write_csv(path: Path, header, rows) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        wr = csv.writer(fh, lineterminator="\n")
        wr.writerow(header)
        wr.writerows([_fmt(v) for v in row] for row in rows)


def export(rep: RunReport, out_dir, request_weighted_hits: bool = False) -> list:
    """requests.csv, cdf_ttft.csv, cdf_tpot.csv, hit_timeline.csv, imbalance.csv,
    detector.csv (when enabled) and summary.json (reference metrics.py:399-497)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    c = _cols(rep)
    m_tt, tt = c.ttft_us()
    m_tp, tp = c.tpot_us()
    m_qd = c.fs >= 0

    def opt(mask, vals):
        return [v if k else None for k, v in zip(mask.tolist(), vals.tolist())]

    cols = [c.rid.tolist(), (c.arr.astype(np.float64) / 1e6).tolist(), c.chosen.tolist(), c.cls.tolist(),
            c.inp.tolist(), c.out.tolist(), c.hit_ratio().tolist(),
            opt(m_tt, tt.astype(np.float64) / 1000.0), opt(m_tp, tp / 1000.0),
            opt(m_qd, (c.fs - c.arr).astype(np.float64) / 1000.0),
            opt(c.ft >= 0, c.ft.astype(np.float64) / 1e6), opt(c.fin >= 0, c.fin.astype(np.float64) / 1e6)]
    path = out / "requests.csv"
    _write_csv(path, REQUEST_COLUMNS, zip(*cols))
    written.append(path)

    for name, vals in (("cdf_ttft.csv", np.sort(tt[m_tt].astype(np.float64) / 1000.0)),
                       ("cdf_tpot.csv", np.sort(tp[m_tp] / 1000.0))):
        n = len(vals)
        path = out / name
        _write_csv(path, ("value_ms", "cum_fraction"), zip(vals.tolist(), [(i + 1) / n for i in range(n)]))
        written.append(path)

    path = out / "hit_timeline.csv"
    _write_csv(path, ("window_start_s", "hit_ratio", "hit_tokens", "input_tokens"),
               hit_timeline(rep, request_weighted=request_weighted_hits))
    written.append(path)

    profiles, _ = imbalance_profile(rep)
    path = out / "imbalance.csv"
    _write_csv(path, ("window_start_s", "instance", "prefill_s", "mean_bs"),
               ((p.window_start_s, i, p.prefill_s[i], p.mean_bs[i]) for p in profiles for i in range(rep.n_instances)))
    written.append(path)

    if rep.detector_enabled:
        path = out / "detector.csv"
        _write_csv(path, ("window_start_s", "class_key", "arrival_fraction", "holders", "others", "suspect", "phase"),
                   ((d.window_start_s, d.class_key, d.fraction, d.n_holders, d.n_others, int(d.suspect), d.phase)
                    for d in rep.detector_rows))
        written.append(path)

    path = out / "summary.json"
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(summarize(rep, request_weighted_hits), fh, indent=2, sort_keys=True)
        fh.write("\n")
    written.append(path)
    return written
