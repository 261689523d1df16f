"""Run results: the reference's RunReport surface over columnar device output.

Field names and derived metrics follow reference metrics.py:31-107
(RequestMetrics, StepRecord, RunReport) and policies.py:83-89
(RoutingDecision). The device writes per-request columns; ``requests``,
``steps`` and ``bs_series`` are materialised lazily so a 1M-request replay
does not pay for a million Python objects unless they are asked for.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class RequestMetrics:
    request_id: int
    class_key: int
    arrival_us: int
    chosen_instance: int
    input_tokens: int
    output_tokens: int
    hit_tokens: int
    first_sched_us: int | None = None
    first_token_us: int | None = None
    finish_us: int | None = None

    @property
    def hit_ratio(self) -> float:
        return self.hit_tokens / self.input_tokens

    @property
    def ttft_us(self) -> int | None:
        return None if self.first_token_us is None else self.first_token_us - self.arrival_us

    @property
    def tpot_us(self) -> float | None:
        if self.finish_us is None or self.first_token_us is None or self.output_tokens < 2:
            return None
        return (self.finish_us - self.first_token_us) / (self.output_tokens - 1)

    @property
    def queue_delay_us(self) -> int | None:
        return None if self.first_sched_us is None else self.first_sched_us - self.arrival_us


@dataclass(frozen=True)
class StepRecord:
    instance: int
    start_us: int
    end_us: int
    prefill_us: int


@dataclass(frozen=True)
class RoutingDecision:
    chosen: int
    scores: dict
    filtered: frozenset
    kind: str
    time_us: int


def _opt(v: int):
    return None if v < 0 else int(v)


@dataclass(frozen=True)
class DetectorRow:
    """Per-window detector state of one top class (reference detector.py:140-148)."""
    window_start_s: float
    class_key: int
    fraction: float
    n_holders: int
    n_others: int
    suspect: bool
    phase: int


class RunReport:
    """Result of ``run`` / ``ClusterSim.run_trace``."""

    def __init__(self, policy_kind: str, seed: int, n_instances: int, block_size: int, trace=None,
                 columns: dict | None = None, step_log: np.ndarray | None = None,
                 end_us: int = 0, queued_at_last_arrival: int = 0, hash_trace=None):
        self.policy_kind = policy_kind
        self.seed = seed
        self.n_instances = n_instances
        self.block_size = block_size
        self.detector_rows: list = []
        self.detector_enabled = False
        self.first_violation_us = None
        self.end_us = end_us
        self.queued_at_last_arrival = queued_at_last_arrival
        self._trace = trace
        self._hash_trace = trace if hash_trace is None else hash_trace   # run_trace's own records
        self.columns = columns or {}
        self._step_log = step_log
        self._requests = None
        self._steps = None
        self._bs = None
        self._hash = None
        n = len(trace) if trace is not None else 0
        self.routed = int((self.columns["chosen"] >= 0).sum()) if n else 0
        self.finished = int((self.columns["finish_us"] >= 0).sum()) if n else 0

    # -- columns (numpy) -------------------------------------------------------------
    @property
    def chosen(self) -> np.ndarray:
        return self.columns["chosen"]

    @property
    def hit_tokens(self) -> np.ndarray:
        return self.columns["hit_tokens"]

    # -- reference surface -------------------------------------------------------------
    @property
    def requests(self) -> list[RequestMetrics]:
        if self._requests is None:
            tr, c = self._trace, self.columns
            if tr is None or len(tr) == 0:
                self._requests = []
            else:
                cols = [tr.request_id.tolist(), tr.class_key.tolist(), tr.arrival_us.tolist(),
                        c["chosen"].tolist(), tr.in_tokens.tolist(), tr.out_tokens.tolist(),
                        c["hit_tokens"].tolist(), c["first_sched_us"].tolist(),
                        c["first_token_us"].tolist(), c["finish_us"].tolist()]
                self._requests = [
                    RequestMetrics(a, b, d, e, f, g, h, _opt(i), _opt(j), _opt(k))
                    for a, b, d, e, f, g, h, i, j, k in zip(*cols)
                ]
        return self._requests

    @property
    def steps(self) -> list[StepRecord]:
        if self._steps is None:
            log = self._sorted_log()
            self._steps = [StepRecord(int(r[0]), int(r[1]), int(r[2]), int(r[3])) for r in log]
        return self._steps

    def _sorted_log(self) -> np.ndarray:
        log = self._step_log
        if log is None or len(log) == 0:
            return np.zeros((0, 6), np.int64)
        # sequential loop pop order: (start, instance, step index) -- cluster.py:203-242
        order = np.lexsort((log[:, 5], log[:, 0], log[:, 1]))
        return log[order]

    @property
    def bs_series(self) -> dict[int, list[tuple[int, int]]]:
        if self._bs is None:
            series = {i: [] for i in range(self.n_instances)}
            ev = []
            tr, c = self._trace, self.columns
            if tr is not None and len(tr):
                rb = c.get("route_bs")
                for k in range(len(tr)):
                    if c["chosen"][k] >= 0:
                        ev.append((int(tr.arrival_us[k]), 0, k, int(c["chosen"][k]), int(rb[k])))
            for r in self._sorted_log():
                ev.append((int(r[1]), 1, int(r[5]), int(r[0]), int(r[4])))
            ev.sort()
            for t, _kind, _i, inst, bs in ev:
                series[inst].append((t, bs))
            self._bs = series
        return self._bs

    @property
    def arrivals_hash(self) -> str:
        """sha256 over ``f"{id}:{arrival_us}\\n"`` (reference cluster.py:184-187)."""
        if self._hash is None:
            d = hashlib.sha256()
            tr = self._hash_trace
            if tr is not None:
                for rid, t in zip(tr.request_id.tolist(), tr.arrival_us.tolist()):
                    d.update(f"{rid}:{t}\n".encode())
            self._hash = d.hexdigest()
        return self._hash

    def ttft_series_us(self) -> list[int]:
        return [r.ttft_us for r in self.requests if r.ttft_us is not None]

    def tpot_series_us(self) -> list[float]:
        return [r.tpot_us for r in self.requests if r.tpot_us is not None]

    def cluster_hit_ratio(self, request_weighted: bool = False) -> float | None:
        tr = self._trace
        if tr is None or len(tr) == 0:
            return None
        ht = self.columns["hit_tokens"].astype(np.float64)
        if request_weighted:
            return float(np.mean(ht / tr.in_tokens))
        return float(ht.sum() / tr.in_tokens.sum())


def percentile(values, p: float):
    """Nearest-rank percentile, the ceil(p/100 * n)-th order statistic (reference metrics.py:162-170)."""
    if len(values) == 0:
        raise ValueError("percentile of an empty series")
    if not 0.0 <= p <= 100.0:
        raise ValueError("p must be in [0, 100]")
    xs = sorted(values)
    return xs[max(math.ceil(p / 100.0 * len(xs)), 1) - 1]
