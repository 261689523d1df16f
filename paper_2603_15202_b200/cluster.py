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
from .trace import PackedTrace, TraceRecord, class_key, validate_against_block_size

_POLICY = {"multiplicative": 0, "vllm": 1, "least_bs": 2, "linear": 3, "filter": 4, "simulate": 5}
INT64_MAX = (1 << 63) - 1



def _scores_dict(scores: np.ndarray, skip_nan: bool) -> dict:
    """RoutingDecision.scores (policies.py:84-89) from the device's score buffer: the C helper
    _rsimpy (csrc/rsim_py.c, built by __graft_entry__.build) when present."""
    try:
        from ._rsimpy import scores_dict
    except ImportError:
        if skip_nan:
            return {i: s for i, s in enumerate(scores.tolist()) if s == s}
        return dict(enumerate(scores.tolist()))
    s = np.ascontiguousarray(scores, dtype=np.float64)
    return scores_dict(s.ctypes.data, s.shape[0], skip_nan)

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
    # the tables hold DISTINCT keys: 1.15x the estimated mean per instance (measured max/mean:
    # 1.04 api64, 1.15 chat1024) -- sizing from non-distinct keys made chat1024's tables 10x
    # too large for L2
    # (memoised on the trace: a sizing guess is never a correctness matter -- an underestimate
    # regrows on device, RSIM_E_TABLE_FULL -- and repeated run() calls on one trace skip the sample)
    memo = trace.__dict__.setdefault("_distinct_memo", {})
    dk = memo.get((N, bs))
    if dk is None:
        dk = memo[(N, bs)] = distinct_keys_per_instance(trace, N, bs)
    est = int(1.15 * dk) + maxchain + 128
    cap = config.cache.capacity_blocks
    if cap is not None:
        est = min(est, cap + maxchain + 64)
    est = min(est, total + 64)
    n = len(trace)
    q = min(n + 16, max(256, 4 * n // N + 256))
    return Sizing(q, est, history_capacity(trace, config))


def distinct_keys_per_instance(trace: PackedTrace, n_instances: int, block_size: int,
                               sample: int = 2048) -> float:
    """Mean distinct KV$ keys one instance ends up holding (no eviction), estimated from an evenly
    spaced sample of requests. A chain key lives on every instance a request carrying it was
    routed to, so the (key, instance) pairs are bounded by sum_k min(count_k, N): block hashes
    seen once in the sample are extrapolated as request-private, repeated ones by their scaled
    count (block values stand in for chain keys: equal chain keys have equal blocks). Output-block
    keys are salted by request id (engine.py:363-372), so always private. An underestimate is
    caught on device (RSIM_E_TABLE_FULL) and regrown."""
    R = len(trace)
    off = trace.blk_off
    nb = np.diff(off)
    idx = np.unique(np.linspace(0, R - 1, min(R, sample)).astype(np.int64))
    frac = len(idx) / R
    lens = nb[idx]
    pos = np.repeat(off[idx] - np.concatenate(([0], np.cumsum(lens[:-1]))), lens) + np.arange(int(lens.sum()))
    _, counts = np.unique(trace.blocks[pos], return_counts=True)
    private = int((counts == 1).sum()) / frac
    shared = float(np.minimum(counts[counts > 1] / frac, n_instances).sum())
    out_keys = int(((trace.out_tokens + block_size - 1) // block_size).sum())
    return (private + shared + out_keys) / n_instances


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
        return self.insert_keys(self._sim._device().chain_keys(np.asarray(blocks, dtype=np.uint64)), now_us)

    def insert_keys(self, keys, now_us: int) -> int:
        return self._sim._do(("insert", self._i, np.asarray(keys, dtype=np.uint64).copy(), int(now_us)))

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


@dataclass(frozen=True)
class SlotView:
    """One request on an instance (the reference's ``_Slot``, engine.py:114-145), read from the
    device queue ring / running list."""
    record: TraceRecord
    hit_blocks: int
    hit_tokens: int
    pending: int
    generated: int
    enqueue_us: int
    first_sched_us: int | None
    index: int                       # the request's position among the sim's loaded requests

    @property
    def keys(self) -> list[int]:
        from .hashing import chain_keys
        return chain_keys(self.record.prefix_blocks)


class _InstanceProxy:
    """``sim.instances[i]`` -- read/poke one instance's device state."""

    def __init__(self, sim: "ClusterSim", idx: int):
        self._sim = sim
        self.id = idx
        self.cache = _CacheProxy(sim, idx)

    def _row(self):
        return self._sim._device().instances()[self.id]

    def _slots(self, kind: int) -> tuple:
        sim = self._sim
        h = sim._device()
        rows = h.slots(self.id)
        rows = rows[rows[:, 1] == kind]
        out = []
        for r in rows:
            idx = int(r[0])
            fs = int(h.request_times(idx, 1)[0][0])
            ht = int(h.decisions(idx, 1)[1][0])
            out.append(SlotView(sim._record(idx), int(r[4]), ht, int(r[2]), int(r[3]),
                                int(sim._arrival_us(idx)), fs if fs >= 0 else None, idx))
        return tuple(out)

    @property
    def queue(self) -> tuple:
        """The FIFO queue (engine.py:212), head first."""
        return self._slots(0)

    @property
    def running(self) -> tuple:
        """The running list (engine.py:213), in order."""
        return self._slots(1)

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
        """InstanceSim.enqueue (engine.py:262-289): DuplicateRequestError when this instance
        already holds the request id, before any state changes."""
        sim = self._sim
        live = sim._holders(record.request_id)
        if self.id in live:
            raise DuplicateRequestError(f"request {record.request_id} already present")
        if live:
            sim._shared_ids.add(record.request_id)
        sim._advance_clock(int(now_us), "enqueue()")
        idx = sim._do(("load", PackedTrace.from_records([record]), np.array([now_us], np.int64)))
        ht = sim._do(("enqueue", self.id, idx, int(now_us)))
        sim._by_rid.setdefault(record.request_id, []).append(idx)
        hb = int(sim._read_hit_blocks(idx)) if ht else 0
        return AdmissionInfo(hb, ht, max(record.input_tokens - ht, 1))


class _StepLogOverflow(Exception):
    def __init__(self, needed: int):
        super().__init__(needed)
        self.needed = needed


def _max_sizing(a: Sizing, b: Sizing) -> Sizing:
    return Sizing(max(a.queue_capacity, b.queue_capacity), max(a.expected_keys, b.expected_keys),
                  max(a.history_capacity, b.history_capacity))


class _HandlePool:
    """Device handles of closed ClusterSims, reused (after rsim_reset) by the next ClusterSim with
    the same native configuration -- the CUDA allocations of a 100k-request replay are not
    repeated for every ``run()``, like a caching allocator. Bounded: at most ``limit`` idle
    handles."""

    def __init__(self, limit: int = 2):
        self.limit = limit
        self.idle: list[tuple[bytes, _native.Handle]] = []

    def take(self, cfg: _native.Config) -> _native.Handle | None:
        key = bytes(cfg)
        for i, (k, h) in enumerate(self.idle):
            if k == key:
                del self.idle[i]
                h.reset()
                return h
        return None

    def give(self, h: _native.Handle) -> None:
        self.idle.append((bytes(h.cfg), h))
        while len(self.idle) > self.limit:
            self.idle.pop(0)[1].close()

    def clear(self) -> None:
        while self.idle:
            self.idle.pop()[1].close()


_POOL = _HandlePool()
# sizes a ClusterSim had to grow to, keyed by the native config it started from
_LEARNED: dict[bytes, tuple[Sizing, int]] = {}


def release_pool() -> None:
    """Free the device memory of idle pooled handles."""
    _POOL.clear()


class ClusterSim:
    """A cluster of instances plus one global routing policy, on the GPU.

    State persists across calls exactly as in the reference: ``route`` / ``enqueue`` /
    ``cache.insert`` calls and successive ``run_trace`` calls all act on the same instances,
    caches and TieBreaker counter, and each ``run_trace`` report covers every request routed
    so far (the reference's Collector, cluster.py:98-101). The state-changing calls are logged
    so that a device ring or table that turns out too small is regrown by replaying them onto
    a larger handle (the device state is a pure function of the calls)."""

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
        self._sizing = sizing_for(None, config)
        self._log_cap = 1 << 16 if record_steps else 0
        self._ops: list = []                  # state-changing calls, replayed onto a regrown handle
        self._stateful = False                # any logged call other than a trace load
        self._log_read = None                 # the step log read by the last run op
        self._det_tracks: dict[int, int] = {}  # route() with the detector: class key -> track
        self._shared_ids: set[int] = set()     # request ids routed / enqueued while live elsewhere
        self._parts: list[PackedTrace] = []   # loaded requests, in load order
        self._arrival: list[np.ndarray] = []  # their arrival (route / enqueue time) in us
        self._reported: list[np.ndarray] = []  # which of them the Collector reports (route / trace)
        self._pending: list = []              # route() records not folded into _parts yet
        self._n = 0
        self._by_rid: dict[int, list[int]] = {}   # request id -> loaded indices (duplicate checks)
        self._runs = 0
        self._first_key: bytes | None = None
        self._clock = 0                       # simulated time reached by the calls so far
        self.instances = [_InstanceProxy(self, i) for i in range(config.n_instances)]

    # -- device handle -----------------------------------------------------------------
    def _native_cfg(self, sizing: Sizing, log_cap: int) -> _native.Config:
        return native_config(self.config, sizing, device=self.device, record_steps=self.record_steps,
                             step_log_capacity=log_cap, ctas=self._shape[0], warps_per_cta=self._shape[1])

    def _device(self) -> _native.Handle:
        if self._handle is None:
            cfg = self._native_cfg(self._sizing, self._log_cap)
            if self._first_key is None:
                self._first_key = bytes(cfg)
                if self._first_key in _LEARNED:
                    self._sizing, self._log_cap = _LEARNED[self._first_key]
                    cfg = self._native_cfg(self._sizing, self._log_cap)
            self._handle = _POOL.take(cfg) or _native.Handle(cfg)
        return self._handle

    def close(self) -> None:
        """Release the device state (the handle returns to the pool for the next ClusterSim)."""
        if self._handle is not None:
            _POOL.give(self._handle)
            self._handle = None

    def _rebuild(self, sizing: Sizing | None = None, log_cap: int | None = None) -> None:
        """A larger handle with every logged call replayed onto it."""
        if self._handle is not None:
            self._handle.close()
            self._handle = None
        if sizing is not None:
            self._sizing = _max_sizing(self._sizing, sizing)
        elif log_cap is None:
            self._sizing = self._sizing.grown()
        if log_cap is not None:
            self._log_cap = max(self._log_cap, log_cap)
        if self._first_key is not None:          # later sims of this shape start at the grown size
            _LEARNED[self._first_key] = (self._sizing, self._log_cap)
        stateful = False
        for op, raised in self._ops:
            try:
                self._exec(op, replaying=True, stateful=stateful)
            except raised or ():
                pass
            stateful = stateful or op[0] != "load"

    def _do(self, op, expected: tuple = ()):
        """Run a state-changing call, regrowing on a capacity signal; log it (with the exception
        it raised, when that exception is part of the reference semantics)."""
        stateful = self._stateful
        for _attempt in range(8):
            try:
                res = self._exec(op, stateful=stateful)
            except _native.CapacityError:
                self._rebuild()
                continue
            except _StepLogOverflow as exc:
                self._rebuild(log_cap=exc.needed + 1024)
                continue
            except expected as exc:
                self._log(op, type(exc))
                raise
            self._log(op, None)
            return res
        raise RuntimeError("device capacities kept overflowing")

    def _log(self, op, raised) -> None:
        self._ops.append((op, raised))
        self._stateful = self._stateful or op[0] != "load"

    def _exec(self, op, *, replaying: bool = False, stateful: bool = False):
        h = self._device()
        kind = op[0]
        if kind == "load":
            _, tr, arr = op
            h.load(arr, tr.in_tokens, tr.out_tokens, tr.request_id, tr.blk_off, tr.blocks)
            if replaying:                 # the bookkeeping of a logged load exists already
                return None
            self._flush()
            first = self._n
            self._parts.append(tr)
            self._arrival.append(np.asarray(arr, np.int64))
            self._reported.append(np.zeros(len(tr), bool))
            self._n += len(tr)
            return first
        if kind == "route":
            _, idx, now, holders = op
            return h.route_one(idx, now, holders=holders)
        if kind == "route_request":       # load + decide in one device call (rsim_route_request)
            _, rec, now, holders, det = op
            if det is not None:
                h.detector_next(*det)
            res = h.route_request(now, rec.input_tokens, rec.output_tokens, rec.request_id, rec.prefix_blocks,
                                  holders=holders)
            return res + (h.last_branch,)
        if kind == "enqueue":
            _, inst, idx, now = op
            return h.enqueue(inst, idx, now)
        if kind == "insert":
            _, inst, keys, now = op
            return h.cache_insert_keys(inst, keys, now)
        if kind == "run":
            # run_trace's loops start with no step scheduled (cluster.py:210-211, 247); a fresh
            # handle has none anyway
            _, first, count, det = op
            if stateful:
                h.unschedule()
            if det is not None:
                h.load_detector(*det)
            if count:
                h.replay(first, count)
            # queued_at_last_arrival (cluster.py:222-223, 277-278): right after the last decision
            queued = int(h.instances()[:, 1].sum()) if count else 0
            h.drain(INT64_MAX)
            if self.record_steps:
                log, needed = h.step_log()
                if log is None:
                    raise _StepLogOverflow(needed)
                self._log_read = log                  # _report's copy (the log is read once per run)
            return queued
        raise ValueError(kind)

    # -- API-mode helpers -------------------------------------------------------------------
    def _flush(self) -> None:
        """Fold the records route() appended since the last fold into the loaded parts."""
        if self._pending:
            recs = [r for r, _, _ in self._pending]
            self._parts.append(PackedTrace.from_records(recs))
            self._arrival.append(np.fromiter((t for _, t, _ in self._pending), np.int64, len(recs)))
            self._reported.append(np.fromiter((ok for _, _, ok in self._pending), bool, len(recs)))
            self._pending = []

    def _record(self, idx: int) -> TraceRecord:
        self._flush()
        for tr in self._parts:
            if idx < len(tr):
                return tr.record(idx)
            idx -= len(tr)
        raise IndexError(idx)

    def _arrival_us(self, idx: int) -> int:
        self._flush()
        for a in self._arrival:
            if idx < len(a):
                return int(a[idx])
            idx -= len(a)
        raise IndexError(idx)

    def _mark_reported(self, idx: int, n: int = 1) -> None:
        self._flush()
        base = 0
        for m in self._reported:
            if base <= idx < base + len(m):
                m[idx - base: idx - base + n] = True
                return
            base += len(m)

    def _holders(self, request_id: int) -> set[int]:
        """Instances where the request id is present (InstanceSim._present: enqueued, not finished)."""
        h = self._device()
        out = set()
        for idx in self._by_rid.get(request_id, ()):
            ch, _ = h.decisions(idx, 1)
            fin = h.request_times(idx, 1)[2]
            if ch[0] >= 0 and fin[0] < 0:
                out.add(int(ch[0]))
        return out

    def _read_hit_blocks(self, idx: int) -> int:
        rec = self._record(idx)
        _, ht = self._device().decisions(idx, 1)
        return min(-(-int(ht[0]) // self.block_size), len(rec.prefix_blocks))

    def _advance_clock(self, now_us: int, what: str) -> None:
        """The device keeps the router view live (indicators.snapshot at staleness 0 equals the
        flushed view while time does not go backwards); a call earlier than the time the sim has
        reached would read the reference's view history instead, which the device path does not
        keep -- refused loudly rather than answered differently."""
        if now_us < self._clock:
            from .config import UnsupportedConfigError
            raise UnsupportedConfigError(f"{what} at {now_us} us precedes the simulated time already reached "
                                         f"({self._clock} us): the device path needs non-decreasing time across calls")
        self._clock = now_us

    def _grow_for(self, trace: PackedTrace | None) -> None:
        need = sizing_for(trace, self.config) if trace is not None and len(trace) else None
        if need is not None and self._handle is None and not self._ops:
            self._sizing = need                  # a fresh sim sizes from its first trace
            return
        if need is not None and (need.queue_capacity > self._sizing.queue_capacity or
                                 need.expected_keys > self._sizing.expected_keys or
                                 need.history_capacity > self._sizing.history_capacity):
            if self._handle is None:
                self._sizing = _max_sizing(self._sizing, need)
            else:
                self._rebuild(need)

    # -- one routing decision (cluster.py:130-154) ---------------------------------------
    def route(self, record: TraceRecord, now_us: int) -> RoutingDecision:
        """Snapshot, score, enqueue on the winner. A request id already present on the chosen
        instance raises DuplicateRequestError after the decision (the TieBreaker counter moved),
        as InstanceSim.enqueue does (engine.py:266-267)."""
        now_us = int(now_us)
        self._advance_clock(now_us, "route()")
        holders = tuple(sorted(self._holders(record.request_id))) if record.request_id in self._by_rid else ()
        idx = self._n
        if self.config.detector is not None and self._runs:
            # (the device detector's tracks of a replayed trace are numbered by that trace and
            # its window was closed by the report's finalize: not continued call by call)
            from .config import UnsupportedConfigError
            raise UnsupportedConfigError("route() with the hotspot detector after a run_trace() on the same ClusterSim")
        det = self._det_class(record, now_us) if self.config.detector is not None else None
        try:
            chosen, _ht, scores, branch = self._do(("route_request", record, now_us, holders, det),
                                                   expected=(DuplicateRequestError,))
        except DuplicateRequestError:
            self._routed(record, now_us, idx, observed=False)
            raise
        self._routed(record, now_us, idx)
        if holders:                               # the id is now live on several instances at once
            self._shared_ids.add(record.request_id)
        kind = self.config.policy.kind
        if branch == 3:                           # verdict force_least_bs (policies.py:228-229)
            kind = "least_bs"
        if branch in (2, 4):                      # holders excluded: scores over the kept candidates only
            excl = np.isnan(scores)
            return RoutingDecision(chosen=chosen, scores=_scores_dict(scores, True),
                                   filtered=frozenset(np.flatnonzero(excl).tolist()), kind=kind, time_us=now_us)
        return RoutingDecision(chosen=chosen, scores=_scores_dict(scores, False),
                               filtered=frozenset(), kind=kind, time_us=now_us)

    def _det_class(self, record: TraceRecord, now_us: int):
        """route() with the detector: the request's track (dense by first arrival, the order
        Detector.observe creates tracks, detector.py:303-307), exemplar length and class key
        (detector.py:41-45, 296-297), and the rows to keep room for (one per top class per window
        roll, detector.py:350-372)."""
        det = self.config.detector
        ck = class_key(record.prefix_blocks, det.class_key_blocks)
        t = self._det_tracks.get(ck)
        if t is None:                 # (registered when the call succeeds: a failed call creates none)
            t = len(self._det_tracks)
        rows = (int(now_us / 1e6 / det.window_s) + 3) * det.top_k_classes
        return (t, min(det.class_key_blocks, len(record.prefix_blocks)), ck, rows)

    def _routed(self, record: TraceRecord, now_us: int, idx: int, observed: bool = True) -> None:
        """Bookkeeping of a routed record (loaded on the device either way). A duplicate
        (observed=False) was decided but never enqueued: the Collector does not report it and
        it is present nowhere (cluster.py:140-152, engine.py:266-267)."""
        if self.config.detector is not None and observed:
            self._det_tracks.setdefault(class_key(record.prefix_blocks, self.config.detector.class_key_blocks),
                                        len(self._det_tracks))
        self._pending.append((record, now_us, observed))
        self._n += 1
        if observed:
            self._by_rid.setdefault(record.request_id, []).append(idx)

    # -- trace replay (cluster.py:172-201) -----------------------------------------------------
    def run_trace(self, records: Sequence[TraceRecord] | PackedTrace) -> RunReport:
        self._flush()
        trace = PackedTrace.from_records(records)
        validate_against_block_size(trace, self.block_size)
        if len(trace):
            if np.unique(trace.request_id).shape[0] != len(trace):
                raise ValueError("duplicate request id in trace")
            if (np.diff(trace.arrival_s) < 0).any():
                raise ValueError("trace arrivals are not sorted")
        det = self.config.detector
        if det is not None and self._ops:
            from .config import UnsupportedConfigError
            raise UnsupportedConfigError("the hotspot detector replays one trace per ClusterSim on the device")
        if len(trace) and self._by_rid and any(self._holders(int(r)) for r in trace.request_id
                                               if int(r) in self._by_rid):
            from .config import UnsupportedConfigError
            raise UnsupportedConfigError("trace request ids still present from earlier route()/enqueue() calls")
        if self._shared_ids and any(self._holders(r) for r in self._shared_ids):
            # the reference's Collector keeps one entry per id for events (metrics.py:116-139): the
            # steps of every live copy would report into the newest copy's RequestMetrics, which
            # the per-copy device columns do not reproduce -- refused rather than answered differently
            from .config import UnsupportedConfigError
            raise UnsupportedConfigError("run_trace() while a request id is live on several instances "
                                         "(route()/enqueue() of an id already present elsewhere)")
        if len(trace) and self._ops:
            self._advance_clock(int(trace.arrival_us[0]), "run_trace()'s first arrival")
        fresh = not self._ops
        self._grow_for(trace if fresh else _concat_all(self._parts + [trace]))
        if self.record_steps:
            need = self._log_cap_for(trace)
            if need > self._log_cap:
                if self._handle is None:
                    self._log_cap = need
                else:
                    self._rebuild(log_cap=need)
        n = len(trace)
        first = self._do(("load", trace, trace.arrival_us)) if n else self._n
        if n:
            self._mark_reported(first, n)
        dl = None
        if det is not None and n:
            tid, ex_off, ex_len, ckey = detector_classes(trace, det.class_key_blocks)
            windows = int(trace.arrival_us[-1] / 1e6 / det.window_s) + 3
            dl = (tid, ex_off, ex_len, ckey, windows * det.top_k_classes + det.top_k_classes)
        queued_last = self._do(("run", first, n, dl))
        self._runs += 1
        rep = self._report(trace, queued_last)
        self._clock = max(self._clock, rep.end_us)
        return rep

    def _log_cap_for(self, trace: PackedTrace) -> int:
        n = self._n + len(trace)
        out = int(trace.out_tokens.sum()) + sum(int(p.out_tokens.sum()) for p in self._parts)
        return max(1 << 16, 8 * n + out // 2)

    def _report(self, trace: PackedTrace, queued_last: int) -> RunReport:
        self._flush()
        h = self._device()
        N = self._n
        inst = h.instances()
        last = int(trace.arrival_us[-1]) if len(trace) else 0
        end_us = int(max(last, int(inst[:, 10].max()) if N else 0))
        cols = {}
        rep_mask = np.concatenate(self._reported) if self._reported else np.zeros(0, bool)
        alltr = _concat_all(self._parts) if self._parts else None
        if N:
            ch, ht = h.decisions(0, N)
            fs, ft, fin = h.request_times(0, N)
            bs = h.route_bs(0, N)
            full = {"chosen": ch, "hit_tokens": ht, "first_sched_us": fs, "first_token_us": ft,
                    "finish_us": fin, "route_bs": bs}
            cols = {k: v[rep_mask] for k, v in full.items()}
            alltr = _with_arrival(alltr, np.concatenate(self._arrival))
            alltr = _take(alltr, np.flatnonzero(rep_mask))
        log = None
        if self.record_steps:
            log = self._log_read if self._log_read is not None else h.step_log()[0]
            self._log_read = None
        rep = RunReport(self.config.policy.kind, self.config.seed, self.config.n_instances, self.block_size,
                        trace=alltr, columns=cols, step_log=log, end_us=end_us,
                        queued_at_last_arrival=queued_last, hash_trace=trace)
        if self.config.detector is not None:              # cluster.py:194-201
            rep.detector_enabled = True
            if len(trace):
                h.detector_finalize()
                rows, rep.first_violation_us = h.read_detector()
                rep.detector_rows = [DetectorRow(*r) for r in rows]
        return rep


def _concat_all(parts: list[PackedTrace]) -> PackedTrace:
    from .trace import concat_packed
    return parts[0] if len(parts) == 1 else concat_packed(parts)


def _with_arrival(tr: PackedTrace, arrival_us: np.ndarray) -> PackedTrace:
    """The loaded requests as the Collector saw them: arrival = the route / enqueue time."""
    if np.array_equal(tr.arrival_us, arrival_us):
        return tr
    out = PackedTrace(tr.request_id, tr.arrival_s, tr.in_tokens, tr.out_tokens, tr.class_key, tr.blk_off, tr.blocks)
    out.arrival_us = np.asarray(arrival_us, np.int64)
    return out


def _take(tr: PackedTrace, idx: np.ndarray) -> PackedTrace:
    if idx.size == len(tr):
        return tr
    B = np.diff(tr.blk_off)[idx]
    off = np.zeros(idx.size + 1, np.int64)
    np.cumsum(B, out=off[1:])
    blocks = np.concatenate([tr.blocks[tr.blk_off[i]:tr.blk_off[i + 1]] for i in idx]) if idx.size else tr.blocks[:0]
    out = PackedTrace(tr.request_id[idx], tr.arrival_s[idx], tr.in_tokens[idx], tr.out_tokens[idx],
                      tr.class_key[idx], off, blocks)
    out.arrival_us = tr.arrival_us[idx]
    return out


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
