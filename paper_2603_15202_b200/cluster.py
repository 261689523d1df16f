"""Drop-in ``ClusterSim`` / ``run`` whose routing runs on the B200.

Mirrors the reference scheduler API (reference cluster.py:67-292):

* ``ClusterSim(config)``               -> one librsim handle (device state)
* ``ClusterSim.route(record, now_us)``  -> one fused probe/score/argmin/enqueue
  launch (cluster.py:130-154); engine steps are NOT advanced, as in the
  reference
* ``ClusterSim.run_trace(records)``     -> the whole trace replayed on device
  in one persistent launch (cluster.py:172-201 with the instance-parallel
  loop of :244-287), then the final drain
* ``run(records, config)``              -> ``ClusterSim(config).run_trace``
* ``sim.instances[i].cache.insert / match_prefix`` and
  ``sim.instances[i].enqueue`` poke device state like the reference tests do.

Errors map to the reference's exception types (ValueError, TraceError,
CacheFullError, DuplicateRequestError, InvariantError, NoInstancesError).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .config import ClusterConfig, DuplicateRequestError
from .hashing import MASK64, stable_key
from .report import DetectorRow, RoutingDecision, RunReport
from .trace import PackedTrace, TraceRecord, validate_against_block_size

_POLICY = {"multiplicative": 0, "vllm": 1, "least_bs": 2, "linear": 3, "filter": 4, "simulate": 5}
INT64_MAX = (1 << 63) - 1


def _next_pow2_log2(v: int) -> int:
    return max(0, int(v - 1).bit_length())


@dataclass(frozen=True)
class Sizing:
    """Per-instance device capacities (queue ring, KV$ table)."""
    queue_capacity: int
    expected_keys: int
    history_capacity: int = 0      # view-history ring entries (staleness > 0), 0 = library default

    def grown(self) -> "Sizing":
        return Sizing(self.queue_capacity * 4, self.expected_keys * 4, max(self.history_capacity, 256) * 4)


def sizing_for(trace: PackedTrace | None, config: ClusterConfig) -> Sizing:
    """Size rings/tables from the trace: generous multiples of the per-instance
    average, bounded by the capacity-limited worst case. Too small a guess is
    detected on device (RSIM_E_QUEUE_OVERFLOW / RSIM_E_TABLE_FULL) and the
    replay is rerun larger -- the replay is a pure function of its inputs."""
    N = config.n_instances
    if trace is None or len(trace) == 0:
        return Sizing(1024, 3000)
    bs = config.cache.block_size
    chain = trace.n_blocks + (trace.out_tokens + bs - 1) // bs
    total = int(chain.sum())
    maxchain = int(chain.max())
    est = 4 * total // N + 4 * maxchain + 1024
    cap = config.cache.capacity_blocks
    if cap is not None:
        est = min(est, cap + maxchain + 64)
    est = min(est, total + 64)
    n = len(trace)
    q = min(n + 16, max(256, 4 * n // N + 256))
    return Sizing(q, est, history_capacity(trace, config))


def history_capacity(trace: PackedTrace, config: ClusterConfig) -> int:
    """Live view-history entries one instance may hold (staleness > 0): everything
    appended within one staleness window -- its enqueues (4x the per-instance
    share of the busiest window's arrivals) and its steps (one per minimum step
    cost) -- plus slack. Older entries are dropped on device once no later
    snapshot can see them."""
    stal = staleness_us(config)
    if stal <= 0:
        return 0
    arr = trace.arrival_us
    win = int((np.searchsorted(arr, arr + stal, side="right") - np.arange(len(arr))).max())
    cm = config.cost_model
    min_step = max(1.0, 1000.0 * min(cm.prefill_base_ms + cm.prefill_per_token_ms,
                                     cm.decode_base_ms + cm.decode_per_seq_ms))
    return int(min(win, 4 * win // config.n_instances + 64) + stal / min_step + 64)


def staleness_us(config: ClusterConfig) -> int:
    return int(round(config.staleness_ms * 1000.0))         # cluster.py:77


def native_config(config: ClusterConfig, sizing: Sizing, *, device: int = 0, record_steps: bool = False,
                  step_log_capacity: int = 0, ctas: int = 0, warps_per_cta: int = 0, world: int = 1,
                  rank: int = 0, comm_timeout_ms: int = 20000) -> _native.Config:
    cm, cache, pol = config.cost_model, config.cache, config.policy
    tie = stable_key(config.seed, pol.tie_break_seed)            # cluster.py:90-94
    c = _native.Config()
    c.n_instances = config.n_instances
    c.block_size = cache.block_size
    c.capacity_blocks = -1 if cache.capacity_blocks is None else cache.capacity_blocks
    c.prefill_base_ms = cm.prefill_base_ms
    c.prefill_per_token_ms = cm.prefill_per_token_ms
    c.decode_base_ms = cm.decode_base_ms
    c.decode_per_seq_ms = cm.decode_per_seq_ms
    c.decode_per_ctx_token_ms = cm.decode_per_ctx_token_ms
    c.chunk_tokens = cm.chunk_tokens
    c.max_batch_requests = cm.max_batch_requests
    c.policy = _POLICY[pol.kind]
    c.kv_indicator = 0 if pol.kv_indicator == "p_tokens" else 1
    c.balance_indicator = 0 if pol.balance_indicator == "bs" else 1
    c.debug_checks = int(config.debug_checks)
    c.q_weight = pol.q_weight
    c.tie_seed_lo = tie & MASK64
    c.tie_seed_hi = 0
    c.device = device
    c.queue_capacity = sizing.queue_capacity
    c.table_slots_log2 = 0
    c.expected_keys = sizing.expected_keys
    c.ctas = ctas
    c.warps_per_cta = warps_per_cta
    c.record_steps = int(record_steps)
    c.step_log_capacity = step_log_capacity
    c.world = world
    c.rank = rank
    c.comm_timeout_ms = comm_timeout_ms
    c.kv_weight = pol.kv_weight
    c.bs_norm_cap = float(pol.bs_norm_cap) if pol.bs_norm_cap is not None else 0.0
    c.range_threshold = pol.range_threshold
    c.staleness_us = staleness_us(config)
    c.history_capacity = sizing.history_capacity
    # Policy.sim_cost_model (policies.py:206-211): the TTFT replay's coefficients
    scm = cm.scaled(pol.mis_tuned_factor) if pol.mis_tuned else cm
    c.sim_prefill_base_ms = scm.prefill_base_ms
    c.sim_prefill_per_token_ms = scm.prefill_per_token_ms
    c.sim_decode_base_ms = scm.decode_base_ms
    c.sim_decode_per_seq_ms = scm.decode_per_seq_ms
    c.sim_decode_per_ctx_token_ms = scm.decode_per_ctx_token_ms
    det = config.detector
    if det is not None:
        c.det_on = 1
        c.det_top_k_classes = det.top_k_classes
        c.det_class_key_blocks = det.class_key_blocks
        c.det_mitigation = 1 if det.mitigation == "force_least_bs" else 0
        c.det_compare_mean_non_holder = int(bool(det.compare_mean_non_holder))
        c.det_window_s = float(det.window_s)
        c.det_consecutive_multiplier = float(det.consecutive_multiplier)
    return c


def detector_classes(trace: PackedTrace, key_blocks: int):
    """Dense class tracks of a trace for the device detector: per request its track
    (numbered by first arrival, the order Detector.observe creates them,
    detector.py:303-307); per track the exemplar -- the first request's leading
    min(key_blocks, B) chain keys (offset, length) -- and the class key
    (detector.py:41-45)."""
    from .hashing import GOLDEN64, combine64, combine64_np
    from .trace import CLASS_SALT
    B = np.diff(trace.blk_off)
    if (B < 1).any():
        raise ValueError("class_key needs at least one block")
    acc = np.full(len(trace), combine64(GOLDEN64, CLASS_SALT), np.uint64)
    for j in range(key_blocks):
        m = B > j
        acc[m] = combine64_np(acc[m], trace.blocks[trace.blk_off[:-1][m] + j])
    keys, first, inv = np.unique(acc, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")              # classes by first arrival
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    tid = rank[inv.ravel()].astype(np.int32)
    fr = first[order]
    return tid, trace.blk_off[:-1][fr].astype(np.int64), np.minimum(B[fr], key_blocks).astype(np.int32), keys[order]


@dataclass(frozen=True)
class AdmissionInfo:          # engine.py:147-151
    hit_blocks: int
    hit_tokens: int
    pending_prefill: int


class _CacheProxy:
    """``inst.cache`` -- the instance's device-resident PrefixCache."""

    def __init__(self, sim: "ClusterSim", idx: int):
        self._sim, self._i = sim, idx

    def insert(self, blocks, now_us: int) -> int:
        h = self._sim._device()
        return h.cache_insert_keys(self._i, h.chain_keys(np.asarray(blocks, dtype=np.uint64)), now_us)

    def insert_keys(self, keys, now_us: int) -> int:
        return self._sim._device().cache_insert_keys(self._i, keys, now_us)

    def match_prefix(self, blocks) -> int:
        h = self._sim._device()
        return h.cache_match_keys(self._i, h.chain_keys(np.asarray(blocks, dtype=np.uint64)))

    def match_keys(self, keys) -> int:
        return self._sim._device().cache_match_keys(self._i, keys)

    @property
    def occupancy(self) -> int:
        return int(self._sim._device().instances()[self._i, 11])

    @property
    def capacity_blocks(self):
        return self._sim.config.cache.capacity_blocks


class _InstanceProxy:
    """``sim.instances[i]`` -- read/poke one instance's device state."""

    def __init__(self, sim: "ClusterSim", idx: int):
        self._sim = sim
        self.id = idx
        self.cache = _CacheProxy(sim, idx)

    def _row(self):
        return self._sim._device().instances()[self.id]

    @property
    def queue(self):
        return tuple(range(int(self._row()[1])))

    @property
    def running(self):
        return tuple(range(int(self._row()[0])))

    @property
    def busy_until_us(self) -> int:
        return int(self._row()[10])

    @property
    def block_size(self) -> int:
        return self._sim.block_size

    def view(self):
        """Router-visible (r, q, pending, total, dc) (engine.py:226)."""
        return tuple(int(x) for x in self._row()[5:10])

    def enqueue(self, record: TraceRecord, now_us: int, keys=None) -> AdmissionInfo:
        sim = self._sim
        idx = sim._append(record)
        ht = sim._device().enqueue(self.id, idx, now_us)
        hb = int(sim._read_hit_blocks(idx)) if ht else 0
        return AdmissionInfo(hb, ht, max(record.input_tokens - ht, 1))


class _StepLogOverflow(Exception):
    def __init__(self, needed: int):
        super().__init__(needed)
        self.needed = needed


class ClusterSim:
    """A cluster of instances plus one global routing policy, on the GPU."""

    def __init__(self, config: ClusterConfig, *, device: int = 0, record_steps: bool = True,
                 ctas: int = 0, warps_per_cta: int = 0):
        config.validate()
        config.check_device_supported()
        self.config = config
        self.block_size = config.cache.block_size
        self.staleness_us = round(config.staleness_ms * 1000.0)
        self.device = device
        self.record_steps = record_steps
        self._shape = (ctas, warps_per_cta)
        self._handle: _native.Handle | None = None
        self._api_records: list[TraceRecord] = []
        self._present: dict[int, int] = {}
        self.instances = [_InstanceProxy(self, i) for i in range(config.n_instances)]

    # -- device handle -----------------------------------------------------------------
    def _make(self, sizing: Sizing, log_cap: int = 0) -> _native.Handle:
        cfg = native_config(self.config, sizing, device=self.device, record_steps=self.record_steps,
                            step_log_capacity=log_cap, ctas=self._shape[0], warps_per_cta=self._shape[1])
        return _native.Handle(cfg)

    def _device(self) -> _native.Handle:
        if self._handle is None:
            self._handle = self._make(sizing_for(None, self.config))
        return self._handle

    def close(self) -> None:
        if self._handle is not None:
            self._handle.close()
            self._handle = None

    # -- API-mode helpers -------------------------------------------------------------------
    def _append(self, record: TraceRecord) -> int:
        h = self._device()
        tr = PackedTrace.from_records([record])
        h.load(tr.arrival_us, tr.in_tokens, tr.out_tokens, tr.request_id, tr.blk_off, tr.blocks)
        self._api_records.append(record)
        return len(self._api_records) - 1

    def _read_hit_blocks(self, idx: int) -> int:
        rec = self._api_records[idx]
        _, ht = self._device().decisions(idx, 1)
        return min(-(-int(ht[0]) // self.block_size), len(rec.prefix_blocks))

    # -- one routing decision (cluster.py:130-154) ---------------------------------------
    def route(self, record: TraceRecord, now_us: int) -> RoutingDecision:
        prior = self._present.get(record.request_id)
        if prior is not None:
            _, _, fin = self._device().request_times(prior, 1)
            if fin[0] < 0:
                raise DuplicateRequestError(f"request {record.request_id} already present")
        idx = self._append(record)
        chosen, _ht, scores = self._device().route_one(idx, now_us)
        self._present[record.request_id] = idx
        return RoutingDecision(chosen=chosen, scores={i: float(s) for i, s in enumerate(scores)},
                               filtered=frozenset(), kind=self.config.policy.kind, time_us=now_us)

    # -- trace replay (cluster.py:172-201) -----------------------------------------------------
    def run_trace(self, records: Sequence[TraceRecord] | PackedTrace) -> RunReport:
        trace = PackedTrace.from_records(records)
        validate_against_block_size(trace, self.block_size)
        if len(trace):
            if np.unique(trace.request_id).shape[0] != len(trace):
                raise ValueError("duplicate request id in trace")
            if (np.diff(trace.arrival_s) < 0).any():
                raise ValueError("trace arrivals are not sorted")
        if self._api_records:
            raise NotImplementedError("run_trace after route()/enqueue() API calls on the same ClusterSim")
        sizing = sizing_for(trace, self.config)
        n = len(trace)
        log_cap = max(1 << 16, 8 * n + int(trace.out_tokens.sum()) // 2) if self.record_steps else 0
        for _attempt in range(6):
            try:
                return self._replay(trace, sizing, log_cap)
            except _native.CapacityError:
                self.close()
                sizing = sizing.grown()
            except _StepLogOverflow as exc:
                self.close()
                log_cap = exc.needed + 1024
        raise RuntimeError("device capacities kept overflowing")

    def _replay(self, trace: PackedTrace, sizing: Sizing, log_cap: int) -> RunReport:
        n = len(trace)
        if self._handle is None:
            self._handle = self._make(sizing, log_cap)
        h = self._handle
        h.reset()
        queued_last = 0
        if n:
            h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off,
                   trace.blocks)
            det = self.config.detector
            if det is not None:
                tid, ex_off, ex_len, ckey = detector_classes(trace, det.class_key_blocks)
                windows = int(trace.arrival_us[-1] / 1e6 / det.window_s) + 3
                h.load_detector(tid, ex_off, ex_len, ckey, windows * det.top_k_classes + det.top_k_classes)
            h.replay(0, n)
            queued_last = int(h.instances()[:, 1].sum())
        h.drain(INT64_MAX)
        inst = h.instances()
        end_us = int(max(int(trace.arrival_us[-1]) if n else 0, int(inst[:, 10].max()) if n else 0))
        cols = {}
        if n:
            cols["chosen"], cols["hit_tokens"] = h.decisions(0, n)
            cols["first_sched_us"], cols["first_token_us"], cols["finish_us"] = h.request_times(0, n)
            cols["route_bs"] = h.route_bs(0, n)
        log = None
        if self.record_steps:
            log, needed = h.step_log()
            if log is None:
                raise _StepLogOverflow(needed)
        rep = RunReport(self.config.policy.kind, self.config.seed, self.config.n_instances, self.block_size,
                        trace=trace, columns=cols, step_log=log, end_us=end_us,
                        queued_at_last_arrival=queued_last)
        if self.config.detector is not None:              # cluster.py:194-201
            rep.detector_enabled = True
            if n:
                h.detector_finalize()
                rows, rep.first_violation_us = h.read_detector()
                rep.detector_rows = [DetectorRow(*r) for r in rows]
        return rep


def run(records, config: ClusterConfig, **kw) -> RunReport:
    """Simulate a full trace; pure function of (records, config) (cluster.py:290-292)."""
    sim = ClusterSim(config, **kw)
    try:
        return sim.run_trace(records)
    finally:
        sim.close()


def probe_capacity(records, config: ClusterConfig, hi_start: float = 8.0, rate_cap: float = 4096.0,
                   iterations: int = 8, **kw) -> float:
    """Binary-search the highest arrival rate the cluster sustains (reference
    cluster.py:295-330, same search and threshold): a rate is sustainable when the
    queued backlog at the last arrival stays under 2 * n_instances * max_batch_requests.
    Every probe is a full device replay of the rescaled trace (scale_trace)."""
    from .trace import scale_packed
    packed = records if isinstance(records, PackedTrace) else PackedTrace.from_records(list(records))
    limit = 2 * config.n_instances * config.cost_model.max_batch_requests

    def sustainable(rate: float) -> bool:
        return run(scale_packed(packed, rate), config, **kw).queued_at_last_arrival < limit

    lo, hi = 0.0, hi_start
    while sustainable(hi):
        lo = hi
        if hi >= rate_cap:
            return rate_cap
        hi = min(hi * 2.0, rate_cap)
    for _ in range(iterations):
        mid = (lo + hi) / 2.0
        if sustainable(mid):
            lo = mid
        else:
            hi = mid
    return lo
