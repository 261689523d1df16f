"""ctypes binding of librsim (include/rsim.h).

The product path: every routing decision of this package is computed by
librsim's sm_100a kernels. If the library or a suitable GPU is missing,
``lib()`` / ``Handle`` raise -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .config import (CacheFullError, DuplicateRequestError, InvariantError, NoInstancesError,
                     UnsupportedConfigError)
from .trace import TraceError

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSIM_LIB selects an alternate in-tree build (tools/variants.sh experiments)
LIB_PATH = os.environ.get("RSIM_LIB") or os.path.join(_HERE, "librsim.so")

RSIM_OK = 0
E_INVALID, E_TRACE, E_CACHE_FULL, E_DUPLICATE, E_INVARIANT, E_CUDA = 1, 2, 3, 4, 5, 6
E_QUEUE_OVERFLOW, E_TABLE_FULL, E_UNSUPPORTED, E_COMM, E_NO_INSTANCES = 7, 8, 9, 10, 11
E_HISTORY_OVERFLOW = 12


class RsimError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[rsim status {status}] {message}")
        self.status = status


class CapacityError(RsimError):
    """A device ring/table was sized too small; the caller may retry larger."""


_EXC = {
    E_INVALID: ValueError, E_TRACE: TraceError, E_CACHE_FULL: CacheFullError,
    E_DUPLICATE: DuplicateRequestError, E_INVARIANT: InvariantError,
    E_UNSUPPORTED: UnsupportedConfigError, E_NO_INSTANCES: NoInstancesError,
}


RSIM_ABI_VERSION = 2


class Config(C.Structure):
    """rsim_config (include/rsim.h); struct_size / abi_version are filled in on construction."""
    _fields_ = [
        ("struct_size", C.c_uint32), ("abi_version", C.c_uint32),
        ("n_instances", C.c_int32), ("block_size", C.c_int32), ("capacity_blocks", C.c_int64),
        ("prefill_base_ms", C.c_double), ("prefill_per_token_ms", C.c_double),
        ("decode_base_ms", C.c_double), ("decode_per_seq_ms", C.c_double),
        ("decode_per_ctx_token_ms", C.c_double),
        ("chunk_tokens", C.c_int64), ("max_batch_requests", C.c_int64),
        ("policy", C.c_int32), ("kv_indicator", C.c_int32), ("balance_indicator", C.c_int32),
        ("debug_checks", C.c_int32), ("q_weight", C.c_double),
        ("tie_seed_lo", C.c_uint64), ("tie_seed_hi", C.c_uint64),
        ("device", C.c_int32), ("queue_capacity", C.c_int32), ("table_slots_log2", C.c_int32),
        ("ctas", C.c_int32), ("warps_per_cta", C.c_int32), ("record_steps", C.c_int32),
        ("step_log_capacity", C.c_int64), ("expected_keys", C.c_int64),
        ("world", C.c_int32), ("rank", C.c_int32), ("comm_timeout_ms", C.c_int64),
        ("runs_capacity", C.c_int64),
        ("kv_weight", C.c_double), ("bs_norm_cap", C.c_double), ("range_threshold", C.c_int64),
        ("staleness_us", C.c_int64), ("history_capacity", C.c_int32), ("reserved0", C.c_int32),
        ("det_on", C.c_int32), ("det_top_k_classes", C.c_int32), ("det_class_key_blocks", C.c_int32),
        ("det_mitigation", C.c_int32), ("det_compare_mean_non_holder", C.c_int32), ("reserved1", C.c_int32),
        ("det_window_s", C.c_double), ("det_consecutive_multiplier", C.c_double),
        ("sim_prefill_base_ms", C.c_double), ("sim_prefill_per_token_ms", C.c_double),
        ("sim_decode_base_ms", C.c_double), ("sim_decode_per_seq_ms", C.c_double),
        ("sim_decode_per_ctx_token_ms", C.c_double),
    ]

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.struct_size = C.sizeof(Config)
        self.abi_version = RSIM_ABI_VERSION


_lib = None


def lib():
    """Load librsim.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(the router has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, I64, I32 = C.c_void_p, C.c_int64, C.c_int32
    sig = {
        "rsim_create": ([C.POINTER(Config), C.POINTER(C.c_void_p)], C.c_int),
        "rsim_destroy": ([P], None),
        "rsim_last_error": ([P], C.c_char_p),
        "rsim_reset": ([P], C.c_int),
        "rsim_load_trace": ([P, I64, P, P, P, P, P, P], C.c_int),
        "rsim_replay": ([P, I64, I64], C.c_int),
        "rsim_drain": ([P, I64], C.c_int),
        "rsim_read_decisions": ([P, I64, I64, P, P], C.c_int),
        "rsim_read_request_times": ([P, I64, I64, P, P, P], C.c_int),
        "rsim_read_instances": ([P, P], C.c_int),
        "rsim_read_step_log": ([P, P, I64, P], C.c_int),
        "rsim_read_route_bs": ([P, I64, I64, P], C.c_int),
        "rsim_route_one": ([P, I64, I64, P, P, P], C.c_int),
        "rsim_enqueue": ([P, I32, I64, I64, P], C.c_int),
        "rsim_cache_insert_keys": ([P, I32, P, I64, I64, P], C.c_int),
        "rsim_cache_match_keys": ([P, I32, P, I64, P], C.c_int),
        "rsim_probe_batch": ([P, I64, I64, P], C.c_int),
        "rsim_chain_keys": ([P, P, I64, P], C.c_int),
        "rsim_last_timings": ([P, P, P, P], C.c_int),
        "rsim_read_decision_ns": ([P, I64, I64, P], C.c_int),
        "rsim_launch_count": ([P], I64),
        "rsim_rerun": ([P, P], C.c_int),
        "rsim_shard_bounds": ([P, P, P], C.c_int),
        "rsim_mailbox": ([P, P], C.c_int),
        "rsim_mailbox_ipc_handle": ([P, P], C.c_int),
        "rsim_set_peer": ([P, I32, P], C.c_int),
        "rsim_open_peer_ipc": ([P, I32, P], C.c_int),
        "rsim_read_counters": ([P, P], C.c_int),
        "rsim_phase_records": ([P, I64], C.c_int),
        "rsim_read_phase_records": ([P, P, I64, P], C.c_int),
        "rsim_read_step_cycles": ([P, P], C.c_int),
        "rsim_read_phase_times": ([P, P, I64], C.c_int),
        "rsim_load_detector": ([P, I64, P, I32, P, P, P, I64], C.c_int),
        "rsim_detector_finalize": ([P], C.c_int),
        "rsim_read_detector": ([P, P, I64, P, P], C.c_int),
        "rsim_detector_debug": ([P, P, I64], C.c_int),
        "rsim_config_size": ([], C.c_size_t),
        "rsim_check_invariants": ([P], C.c_int),
        "rsim_debug_corrupt": ([P, I32, I32], C.c_int),
        "rsim_route_one_excl": ([P, I64, I64, P, I32, P, P, P], C.c_int),
        "rsim_read_slots": ([P, I32, P, I64, P, P], C.c_int),
        "rsim_unschedule": ([P], C.c_int),
        "rsim_route_request": ([P, I64, I64, I64, C.c_uint64, P, I64, P, I32, P, P, P, P], C.c_int),
        "rsim_detector_next": ([P, I32, I32, C.c_uint64, I64], C.c_int),
        "rsim_synth_generate": ([P, I32, C.c_double, C.c_double, C.c_uint64, I64, I32, P, P, P], C.c_int),
        "rsim_synth_read": ([P, P, P, P, P, P, P, P], C.c_int),
        "rsim_synth_device_arrays": ([P, P], C.c_int),
        "rsim_synth_free": ([P], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.rsim_config_size() != C.sizeof(Config):
        raise RuntimeError(f"librsim's rsim_config is {L.rsim_config_size()} bytes, this binding's "
                           f"{C.sizeof(Config)}: rebuild librsim.so from this tree")
    _lib = L
    return L


EXPORTED = ("rsim_create", "rsim_destroy", "rsim_last_error", "rsim_reset", "rsim_load_trace", "rsim_replay",
            "rsim_drain", "rsim_read_decisions", "rsim_read_request_times", "rsim_read_instances",
            "rsim_read_step_log", "rsim_read_route_bs", "rsim_route_one", "rsim_enqueue",
            "rsim_cache_insert_keys", "rsim_cache_match_keys", "rsim_probe_batch", "rsim_chain_keys",
            "rsim_last_timings", "rsim_read_decision_ns", "rsim_launch_count", "rsim_rerun",
            "rsim_read_counters", "rsim_shard_bounds", "rsim_mailbox", "rsim_mailbox_ipc_handle",
            "rsim_set_peer", "rsim_open_peer_ipc", "rsim_load_detector", "rsim_detector_finalize",
            "rsim_read_detector", "rsim_detector_debug", "rsim_config_size", "rsim_check_invariants",
            "rsim_debug_corrupt", "rsim_route_one_excl", "rsim_read_slots", "rsim_unschedule",
            "rsim_route_request", "rsim_detector_next", "rsim_synth_generate", "rsim_synth_read",
            "rsim_synth_device_arrays", "rsim_synth_free")


class SynthClass(C.Structure):
    """rsim_synth_class (include/rsim.h): one ClassSpec (reference trace.py:58-69)."""
    _fields_ = [("weight", C.c_double), ("shared_blocks", C.c_int64), ("suffix_lo", C.c_int64),
                ("suffix_hi", C.c_int64), ("output_lo", C.c_int64), ("output_hi", C.c_int64)]


def synth_generate(spec, device: int = 0):
    """generate_synthetic(spec) on the GPU (rsim_synth_generate): the PackedTrace columns as
    host arrays (request_id, arrival_s, in_tokens, out_tokens, class_key, blk_off, blocks)."""
    L = lib()
    n_cls = len(spec.classes)
    arr = (SynthClass * max(n_cls, 1))()
    for i, c in enumerate(spec.classes):
        arr[i] = SynthClass(float(c.weight), int(c.shared_blocks), int(c.suffix_blocks[0]), int(c.suffix_blocks[1]),
                            int(c.output_tokens[0]), int(c.output_tokens[1]))
    g, n, nb = C.c_void_p(), C.c_int64(), C.c_int64()
    st = L.rsim_synth_generate(C.cast(arr, C.c_void_p), n_cls, float(spec.duration_s), float(spec.mean_rate_rps),
                               int(spec.seed) & ((1 << 64) - 1), int(spec.block_size), device, C.byref(g),
                               C.byref(n), C.byref(nb))
    if st != RSIM_OK:
        msg = L.rsim_last_error(None).decode()
        raise _EXC[st](msg) if st in _EXC else RsimError(st, msg)
    try:
        n, nb = n.value, nb.value
        cols = (np.empty(n, np.uint64), np.empty(n, np.float64), np.empty(n, np.int64), np.empty(n, np.int64),
                np.empty(n, np.uint64), np.empty(n + 1, np.int64), np.empty(nb, np.uint64))
        st = L.rsim_synth_read(g, *[c.ctypes.data_as(C.c_void_p) for c in cols])
        if st != RSIM_OK:
            raise RsimError(st, L.rsim_last_error(None).decode())
        return cols
    finally:
        L.rsim_synth_free(g)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c64(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Handle:
    """Owns one librsim handle (one GPU's instance shard)."""

    def __init__(self, cfg: Config):
        self._L = lib()
        h = C.c_void_p()
        st = self._L.rsim_create(C.byref(cfg), C.byref(h))
        if st != RSIM_OK:
            self._h = None
            self._raise(st, self._L.rsim_last_error(None).decode())
        self._h = h
        self.cfg = cfg
        lo, hi = self.shard_bounds()
        self.lo, self.n_local = lo, hi - lo

    def close(self):
        if getattr(self, "_h", None):
            self._L.rsim_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _raise(self, st: int, msg: str | None = None):
        if msg is None:
            msg = self._L.rsim_last_error(self._h).decode()
        if st in (E_QUEUE_OVERFLOW, E_TABLE_FULL, E_HISTORY_OVERFLOW):
            raise CapacityError(st, msg)
        exc = _EXC.get(st)
        if exc is not None:
            raise exc(msg)
        raise RsimError(st, msg)

    def _ck(self, st: int):
        if st != RSIM_OK:
            self._raise(st)

    # -- calls ------------------------------------------------------------------------
    def reset(self):
        self._ck(self._L.rsim_reset(self._h))

    def load(self, arrival_us, in_tok, out_tok, rid, blk_off, blocks):
        n = len(arrival_us)
        arrays = (_c64(arrival_us, np.int64), _c64(in_tok, np.int64), _c64(out_tok, np.int64),
                  _c64(rid, np.uint64), _c64(blk_off, np.int64), _c64(blocks, np.uint64))
        if arrays[5].size == 0:
            arrays = arrays[:5] + (np.zeros(1, np.uint64),)
        self._ck(self._L.rsim_load_trace(self._h, n, *(_p(a) for a in arrays)))

    def replay(self, first: int, count: int):
        self._ck(self._L.rsim_replay(self._h, first, count))

    def drain(self, until_us: int = (1 << 63) - 1):
        self._ck(self._L.rsim_drain(self._h, until_us))

    def decisions(self, first: int, count: int):
        ch = np.empty(count, np.int32)
        ht = np.empty(count, np.int64)
        self._ck(self._L.rsim_read_decisions(self._h, first, count, _p(ch), _p(ht)))
        return ch, ht

    def request_times(self, first: int, count: int):
        a, b, c = (np.empty(count, np.int64) for _ in range(3))
        self._ck(self._L.rsim_read_request_times(self._h, first, count, _p(a), _p(b), _p(c)))
        return a, b, c

    def route_bs(self, first: int, count: int):
        a = np.empty(count, np.int64)
        self._ck(self._L.rsim_read_route_bs(self._h, first, count, _p(a)))
        return a

    def decision_ns(self, first: int, count: int):
        a = np.empty(count, np.int64)
        self._ck(self._L.rsim_read_decision_ns(self._h, first, count, _p(a)))
        return a

    def instances(self) -> np.ndarray:
        out = np.empty((self.n_local, 12), np.int64)
        self._ck(self._L.rsim_read_instances(self._h, _p(out)))
        return out

    def step_log(self):
        """(records[n, 6], n) -- records is None when the device log overflowed."""
        n = C.c_int64(0)
        self._L.rsim_read_step_log(self._h, None, 0, C.byref(n))
        if n.value > self.cfg.step_log_capacity and self.cfg.step_log_capacity > 0:
            return None, n.value
        out = np.empty((max(n.value, 1), 6), np.int64)
        self._ck(self._L.rsim_read_step_log(self._h, _p(out), n.value, C.byref(n)))
        return out[: n.value], n.value

    def route_one(self, r: int, now_us: int, want_scores: bool = True, holders=()):
        """One route() decision; ``holders``: instances already holding the request id
        (a decision for one of them raises DuplicateRequestError after the tie-break)."""
        ch = np.zeros(1, np.int32)
        ht = np.zeros(1, np.int64)
        sc = np.empty(self.n_local, np.float64) if want_scores else None
        hd = np.asarray(sorted(holders), np.int32)
        self._ck(self._L.rsim_route_one_excl(self._h, r, now_us, _p(hd) if hd.size else None, int(hd.size),
                                             _p(ch), _p(ht), _p(sc)))
        return int(ch[0]), int(ht[0]), sc

    def route_request(self, now_us: int, input_tokens: int, output_tokens: int, request_id: int, blocks,
                      holders=(), want_scores: bool = True):
        """ClusterSim.route of a request not loaded yet: rsim_route_request appends it to the device
        trace and decides it in one call. ``blocks``: u64 array (or sequence) of its block hashes."""
        if isinstance(blocks, np.ndarray) and blocks.dtype == np.uint64:
            b = np.ascontiguousarray(blocks)
        else:
            try:                                  # hashes already in [0, 2^64)
                b = np.array(blocks, dtype=np.uint64)
            except (OverflowError, TypeError, ValueError):
                b = np.fromiter((x & 0xFFFFFFFFFFFFFFFF for x in blocks), np.uint64)
        out = self._rr_out
        sc = np.empty(self.n_local, np.float64) if want_scores else None
        hd = np.asarray(sorted(holders), np.int32) if holders else None
        self._ck(self._L.rsim_route_request(self._h, now_us, input_tokens, output_tokens,
                                            request_id & 0xFFFFFFFFFFFFFFFF, _p(b) if b.size else None, b.size,
                                            _p(hd), 0 if hd is None else int(hd.size), self._rr_ch_p, self._rr_ht_p,
                                            _p(sc), self._rr_br_p))
        return int(out[0][0]), int(out[1][0]), sc

    @property
    def last_branch(self) -> int:
        """The detector verdict the last route_request applied (0 none, 2 holders excluded,
        3 forced least_bs, 4 excluded + route_filter's batch-size branch)."""
        return int(self._rr_out[2][0])

    def detector_next(self, track: int, exemplar_len: int, class_key: int, rows_capacity: int):
        """The class of the request the next route_request appends (route() with a detector)."""
        self._ck(self._L.rsim_detector_next(self._h, track, exemplar_len, class_key & 0xFFFFFFFFFFFFFFFF,
                                            rows_capacity))

    @property
    def _rr_out(self):
        o = getattr(self, "_rr", None)
        if o is None:
            o = self._rr = (np.zeros(1, np.int32), np.zeros(1, np.int64), np.zeros(1, np.int32))
            self._rr_ch_p, self._rr_ht_p, self._rr_br_p = _p(o[0]), _p(o[1]), _p(o[2])
        return o

    def slots(self, instance: int) -> np.ndarray:
        """(n, 8) int64: the FIFO queue then the running list of a local instance (rsim_read_slots)."""
        nq, nr = C.c_int64(), C.c_int64()
        self._ck(self._L.rsim_read_slots(self._h, instance, None, 0, C.byref(nq), C.byref(nr)))
        n = nq.value + nr.value
        out = np.empty((max(n, 1), 8), np.int64)
        self._ck(self._L.rsim_read_slots(self._h, instance, _p(out), n, C.byref(nq), C.byref(nr)))
        return out[:n]

    def unschedule(self):
        self._ck(self._L.rsim_unschedule(self._h))

    def enqueue(self, instance: int, r: int, now_us: int) -> int:
        ht = np.zeros(1, np.int64)
        self._ck(self._L.rsim_enqueue(self._h, instance, r, now_us, _p(ht)))
        return int(ht[0])

    def cache_insert_keys(self, instance: int, keys, now_us: int) -> int:
        k = _c64(keys, np.uint64)
        ev = np.zeros(1, np.int64)
        self._ck(self._L.rsim_cache_insert_keys(self._h, instance, _p(k), k.size, now_us, _p(ev)))
        return int(ev[0])

    def cache_match_keys(self, instance: int, keys) -> int:
        k = _c64(keys, np.uint64)
        hit = np.zeros(1, np.int64)
        self._ck(self._L.rsim_cache_match_keys(self._h, instance, _p(k), k.size, _p(hit)))
        return int(hit[0])

    def probe_batch(self, first: int, count: int) -> np.ndarray:
        out = np.empty((count, self.n_local), np.int32)
        self._ck(self._L.rsim_probe_batch(self._h, first, count, _p(out)))
        return out

    def chain_keys(self, blocks) -> np.ndarray:
        b = _c64(blocks, np.uint64)
        out = np.empty_like(b)
        self._ck(self._L.rsim_chain_keys(self._h, _p(b), b.size, _p(out)))
        return out

    def timings(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._ck(self._L.rsim_last_timings(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def rerun(self) -> float:
        """Resident full replay; returns device milliseconds."""
        ms = C.c_double()
        self._ck(self._L.rsim_rerun(self._h, C.byref(ms)))
        return ms.value

    def phase_records(self, capacity: int):
        """Enable (capacity > 0) per-(decision, warp) phase records of the next replays."""
        self._ck(self._L.rsim_phase_records(self._h, capacity))

    def read_phase_records(self, n: int) -> np.ndarray:
        w = C.c_int32()
        self._ck(self._L.rsim_read_phase_records(self._h, None, 0, C.byref(w)))
        out = np.zeros((n, w.value, 8), np.uint16)
        self._ck(self._L.rsim_read_phase_records(self._h, out.ctypes.data, n, None))
        return out

    def read_phase_times(self, n: int, warps: int) -> np.ndarray:
        out = np.zeros((n, warps + 4), np.uint64)
        self._ck(self._L.rsim_read_phase_times(self._h, out.ctypes.data, n))
        return out

    # -- hotspot detector ----------------------------------------------------------------
    def load_detector(self, track_of_request, exemplar_offset, exemplar_len, class_key, rows_capacity: int):
        tid = np.ascontiguousarray(track_of_request, dtype=np.int32)
        off = np.ascontiguousarray(exemplar_offset, dtype=np.int64)
        ln = np.ascontiguousarray(exemplar_len, dtype=np.int32)
        key = np.ascontiguousarray(class_key, dtype=np.uint64)
        self._ck(self._L.rsim_load_detector(self._h, len(tid), _p(tid), len(off), _p(off), _p(ln), _p(key),
                                            int(rows_capacity)))

    def detector_finalize(self):
        self._ck(self._L.rsim_detector_finalize(self._h))

    def read_detector(self):
        """(rows, first_violation_us): DetectorRow tuples (window_start_s, class_key, fraction,
        n_holders, n_others, suspect, phase) and None or the first phase-1 time."""
        n, fv = C.c_int64(), C.c_int64()
        self._ck(self._L.rsim_read_detector(self._h, None, 0, C.byref(n), C.byref(fv)))
        raw = np.zeros((max(n.value, 1), 7), np.int64)
        self._ck(self._L.rsim_read_detector(self._h, _p(raw), n.value, C.byref(n), C.byref(fv)))
        raw = raw[:n.value]
        f = raw.view(np.float64)
        rows = [(float(f[i, 0]), int(np.uint64(raw[i, 1])), float(f[i, 2]), int(raw[i, 3]), int(raw[i, 4]),
                 bool(raw[i, 5]), int(raw[i, 6])) for i in range(len(raw))]
        return rows, (None if fv.value < 0 else int(fv.value))

    def step_cycles(self) -> np.ndarray:
        out = np.zeros(32, np.int64)
        self._ck(self._L.rsim_read_step_cycles(self._h, out.ctypes.data))
        return out

    def counters(self) -> np.ndarray:
        out = np.zeros(16, np.int64)
        self._ck(self._L.rsim_read_counters(self._h, _p(out)))
        return out

    def shard_bounds(self):
        lo, hi = C.c_int32(), C.c_int32()
        self._ck(self._L.rsim_shard_bounds(self._h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def mailbox(self) -> int:
        p = C.c_void_p()
        self._ck(self._L.rsim_mailbox(self._h, C.byref(p)))
        return p.value

    def mailbox_ipc_handle(self) -> bytes:
        buf = (C.c_ubyte * 64)()
        self._ck(self._L.rsim_mailbox_ipc_handle(self._h, buf))
        return bytes(buf)

    def set_peer(self, rank: int, ptr: int):
        self._ck(self._L.rsim_set_peer(self._h, rank, C.c_void_p(ptr)))

    def open_peer_ipc(self, rank: int, handle: bytes):
        buf = (C.c_ubyte * 64).from_buffer_copy(handle)
        self._ck(self._L.rsim_open_peer_ipc(self._h, rank, buf))

    def check_invariants(self):
        self._ck(self._L.rsim_check_invariants(self._h))

    def debug_corrupt(self, instance: int, what: int):
        self._ck(self._L.rsim_debug_corrupt(self._h, instance, what))

    def launch_count(self) -> int:
        return int(self._L.rsim_launch_count(self._h))
