"""ctypes wrapper around the CPU oracle (``rsim_oracle.c``).

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU "port"
baseline. Importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg; the product package never imports it.

``run_oracle(trace, config)`` replays a PackedTrace under a ClusterConfig
(ours or the reference's: attributes are read by name) and returns the
per-request decisions and timings the reference's ``run()`` produces
(reference cluster.py:290-292).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

POLICY_CODE = {"multiplicative": 0, "vllm": 1, "least_bs": 2, "linear": 3, "filter": 4, "simulate": 5}


class _Cfg(C.Structure):
    _fields_ = [
        ("n_instances", C.c_int32), ("policy", C.c_int32), ("kv_ind", C.c_int32), ("bal_ind", C.c_int32),
        ("block_size", C.c_int64), ("capacity", C.c_int64),
        ("pb", C.c_double), ("pt", C.c_double), ("db", C.c_double), ("ds", C.c_double),
        ("dc", C.c_double), ("q_weight", C.c_double),
        ("chunk", C.c_int64), ("max_batch", C.c_int64),
        ("tie_lo", C.c_uint64), ("tie_hi", C.c_uint64),
        ("kv_weight", C.c_double), ("bs_norm_cap", C.c_double), ("range_threshold", C.c_int64),
        ("staleness_us", C.c_int64),
        ("det_on", C.c_int32), ("det_top_k", C.c_int32), ("det_kb", C.c_int32), ("det_force", C.c_int32),
        ("det_mean", C.c_int32), ("det_pad", C.c_int32), ("det_window_s", C.c_double), ("det_mult", C.c_double),
        ("spb", C.c_double), ("spt", C.c_double), ("sdb", C.c_double), ("sds", C.c_double), ("sdc", C.c_double),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "rsim_oracle.c")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        L.orc_run.restype = C.c_int
        L.orc_run.argtypes = [C.POINTER(_Cfg), C.c_int64] + [P] * 13 + [C.c_int64, P, P, C.c_int64]
        L.orc_cache_new.restype = P
        L.orc_cache_new.argtypes = [C.c_int64]
        L.orc_cache_free.argtypes = [P]
        L.orc_cache_insert.restype = C.c_int64
        L.orc_cache_insert.argtypes = [P, P, C.c_int64, C.c_int64]
        L.orc_cache_match.restype = C.c_int64
        L.orc_cache_match.argtypes = [P, P, C.c_int64]
        L.orc_cache_touch.argtypes = [P, P, C.c_int64, C.c_int64]
        L.orc_cache_pin.argtypes = [P, P, C.c_int64]
        L.orc_cache_unpin.restype = C.c_int
        L.orc_cache_unpin.argtypes = [P, P, C.c_int64]
        L.orc_cache_occupancy.restype = C.c_int64
        L.orc_cache_occupancy.argtypes = [P]
        L.orc_cache_dump.restype = C.c_int64
        L.orc_cache_dump.argtypes = [P, P, C.c_int64]
        L.orc_chain_keys.argtypes = [P, C.c_int64, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _stable_key(*vals: int) -> int:
    m = (1 << 64) - 1

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)

    acc = 0x9E3779B97F4A7C15
    for v in vals:
        acc = mix(acc ^ (v & m))
    return acc


def sim_cost_coefficients(config) -> tuple:
    """Policy.sim_cost_model (policies.py:206-211): CostModel.scaled(mis_tuned_factor)
    (engine.py:70-79) when mis-tuned, else the engine's own coefficients."""
    cm, pol = config.cost_model, config.policy
    f = float(pol.mis_tuned_factor) if getattr(pol, "mis_tuned", False) else None
    c = (cm.prefill_base_ms, cm.prefill_per_token_ms, cm.decode_base_ms, cm.decode_per_seq_ms,
         cm.decode_per_ctx_token_ms)
    return tuple(float(x) * f if f is not None else float(x) for x in c)


def make_cfg(config) -> _Cfg:
    cm, cache, pol = config.cost_model, config.cache, config.policy
    if pol.kind not in POLICY_CODE:
        raise ValueError(f"oracle covers policies {sorted(POLICY_CODE)}, not {pol.kind!r}")
    tie = _stable_key(config.seed, pol.tie_break_seed)
    det = getattr(config, "detector", None)
    dv = (0, 0, 0, 0, 0, 0, 0.0, 0.0) if det is None else (
        1, int(det.top_k_classes), int(det.class_key_blocks), int(det.mitigation == "force_least_bs"),
        int(bool(det.compare_mean_non_holder)), 0, float(det.window_s), float(det.consecutive_multiplier))
    return _Cfg(config.n_instances, POLICY_CODE[pol.kind],
                0 if pol.kv_indicator == "p_tokens" else 1,
                0 if pol.balance_indicator == "bs" else 1,
                cache.block_size, -1 if cache.capacity_blocks is None else cache.capacity_blocks,
                cm.prefill_base_ms, cm.prefill_per_token_ms, cm.decode_base_ms,
                cm.decode_per_seq_ms, cm.decode_per_ctx_token_ms, pol.q_weight,
                cm.chunk_tokens, cm.max_batch_requests, tie, 0,
                float(getattr(pol, "kv_weight", 0.4)),
                float(pol.bs_norm_cap) if getattr(pol, "bs_norm_cap", None) is not None else 0.0,
                int(getattr(pol, "range_threshold", 4)),
                int(round(float(getattr(config, "staleness_ms", 0.0)) * 1000.0)),   # cluster.py:77
                *dv, *sim_cost_coefficients(config))


class OracleError(RuntimeError):
    pass


@dataclass
class OracleResult:
    chosen: np.ndarray
    hit_tokens: np.ndarray
    first_sched_us: np.ndarray
    first_token_us: np.ndarray
    finish_us: np.ndarray
    end_us: int
    queued_at_last_arrival: int
    finished: int
    log: np.ndarray | None  # (n, 6): kind, inst, start, end, prefill_us, bs
    route_ns: np.ndarray | None
    evicted: int = 0
    # detector (None without one): DetectorRow tuples (window_start_s, class_key, fraction,
    # n_holders, n_others, suspect, phase) and first_violation_us
    detector_rows: list | None = None
    first_violation_us: int | None = None


def run_oracle(trace, config, *, with_log: bool = False, time_routes: bool = False,
               _log_cap: int | None = None, _rows_cap: int | None = None) -> OracleResult:
    """Replay ``trace`` (a PackedTrace) on the CPU oracle."""
    L = lib()
    cfg = make_cfg(config)
    R = len(trace)
    arr = np.ascontiguousarray(trace.arrival_us, dtype=np.int64)
    i_in = np.ascontiguousarray(trace.in_tokens, dtype=np.int64)
    i_out = np.ascontiguousarray(trace.out_tokens, dtype=np.int64)
    rid = np.ascontiguousarray(trace.request_id, dtype=np.uint64)
    off = np.ascontiguousarray(trace.blk_off, dtype=np.int64)
    blk = np.ascontiguousarray(trace.blocks, dtype=np.uint64)
    if blk.size == 0:
        blk = np.zeros(1, np.uint64)
    chosen = np.empty(R, np.int32)
    hit = np.empty(R, np.int64)
    fs, ft, fin = (np.empty(R, np.int64) for _ in range(3))
    summary = np.zeros(7, np.int64)
    det_on = getattr(config, "detector", None) is not None
    rows_cap = _rows_cap if _rows_cap is not None else (4096 if det_on else 0)
    rows = np.zeros((max(rows_cap, 1), 7), np.int64)
    log_cap = 0
    log = None
    if with_log:
        log_cap = _log_cap or max(16, 64 * R)
        log = np.empty((log_cap, 6), np.int64)
    rns = np.empty(R, np.int64) if time_routes else None
    rc = L.orc_run(C.byref(cfg), R, _ptr(arr), _ptr(i_in), _ptr(i_out), _ptr(rid), _ptr(off), _ptr(blk),
                   _ptr(chosen), _ptr(hit), _ptr(fs), _ptr(ft), _ptr(fin), _ptr(summary),
                   _ptr(log) if with_log else None, log_cap, _ptr(rns), _ptr(rows), rows_cap)
    if rc == -1:
        raise OracleError("CacheFullError")
    if rc == -4:
        raise ValueError("class_key needs at least one block")
    if rc == -5:
        raise RuntimeError("TTFT replay did not converge")
    if det_on and summary[5] > rows_cap:
        return run_oracle(trace, config, with_log=with_log, time_routes=time_routes, _log_cap=_log_cap,
                          _rows_cap=int(summary[5]))
    if rc != 0:
        raise OracleError(f"oracle error {rc}")
    if with_log:
        n = int(summary[3])
        if n > log_cap:
            return run_oracle(trace, config, with_log=True, time_routes=time_routes, _log_cap=n)
        log = log[:n].copy()
    drows = fv = None
    if det_on:
        r = rows[:int(summary[5])]
        drows = [(float(r[i, 0:1].view(np.float64)[0]), int(np.uint64(r[i, 1])), float(r[i, 2:3].view(np.float64)[0]),
                  int(r[i, 3]), int(r[i, 4]), bool(r[i, 5]), int(r[i, 6])) for i in range(len(r))]
        fv = None if summary[6] < 0 else int(summary[6])
    return OracleResult(chosen, hit, fs, ft, fin, int(summary[0]), int(summary[1]), int(summary[2]), log, rns,
                        int(summary[4]), drows, fv)


class OracleCache:
    """The oracle's PrefixCache (reference kvcache.py) for op-sequence parity tests."""

    def __init__(self, capacity: int | None):
        self._L = lib()
        self._h = self._L.orc_cache_new(-1 if capacity is None else capacity)

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.orc_cache_free(self._h)
            self._h = None

    @staticmethod
    def _k(keys):
        return np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))

    def insert_keys(self, keys, now: int) -> int:
        k = self._k(keys)
        r = self._L.orc_cache_insert(self._h, _ptr(k), k.size, now)
        if r < 0:
            raise OracleError("CacheFullError")
        return r

    def match_keys(self, keys) -> int:
        k = self._k(keys)
        return self._L.orc_cache_match(self._h, _ptr(k), k.size)

    def touch_keys(self, keys, upto: int, now: int) -> None:
        k = self._k(keys)
        self._L.orc_cache_touch(self._h, _ptr(k), upto, now)

    def pin_keys(self, keys, upto: int) -> None:
        k = self._k(keys)
        self._L.orc_cache_pin(self._h, _ptr(k), upto)

    def unpin_keys(self, keys, upto: int) -> None:
        k = self._k(keys)
        if self._L.orc_cache_unpin(self._h, _ptr(k), upto):
            raise ValueError("unpin of a chain that is not pinned")

    @property
    def occupancy(self) -> int:
        return self._L.orc_cache_occupancy(self._h)

    def dump(self) -> dict[int, tuple[int, int, int]]:
        n = self.occupancy
        out = np.empty((max(n, 1), 4), np.int64)
        self._L.orc_cache_dump(self._h, _ptr(out), n)
        return {int(np.uint64(r[0])): (int(r[1]), int(r[2]), int(r[3])) for r in out[:n]}


def chain_keys(blocks) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.uint64))
    out = np.empty_like(b)
    lib().orc_chain_keys(_ptr(b), b.size, _ptr(out))
    return out
