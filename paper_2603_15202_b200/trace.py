"""Request traces: the record type, JSONL I/O, rescaling, the seeded
synthetic generator, and the packed (CSR) form the device consumes.

Semantics follow the reference trace module (``pkg/src/routesim/trace.py``):
record schema ``:42-54``, JSONL format ``:3-9`` / ``:108-182``, rescaling
``:197-213``, generator ``:218-268`` (same ``random.Random`` streams and
``stable_key`` salts, so the same spec yields the same trace), block-count
check ``:271-281``. The generator is vectorised with numpy where the
reference loops over ``stable_key`` per block.
"""

from __future__ import annotations

import dataclasses
import json
import math
import os
import random
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

from .hashing import MASK64, stable_key, stable_key_np

SHARED_SALT = 0x5EED_0001
SUFFIX_SALT = 0x5EED_0002
CLASS_RNG_SALT = 0x5EED_0003
CLASS_SALT = 0xC1A5_5000  # detector.py:38


class TraceError(Exception):
    """Malformed or inconsistent trace input (``line`` is 1-based if known)."""

    def __init__(self, message: str, line: int | None = None) -> None:
        super().__init__(message if line is None else f"line {line}: {message}")
        self.line = line


@dataclass(frozen=True)
class TraceRecord:
    request_id: int
    arrival_s: float
    prefix_blocks: tuple[int, ...]
    input_tokens: int
    output_tokens: int
    class_key: int


@dataclass(frozen=True)
class ClassSpec:
    weight: float
    shared_blocks: int
    suffix_blocks: tuple[int, int] = (2, 4)
    output_tokens: tuple[int, int] = (32, 64)


@dataclass(frozen=True)
class SyntheticSpec:
    duration_s: float
    mean_rate_rps: float
    classes: tuple[ClassSpec, ...]
    seed: int = 0
    block_size: int = 16

    def validate(self) -> None:
        if self.duration_s <= 0 or self.mean_rate_rps <= 0 or self.block_size < 1:
            raise TraceError("duration, rate, and block size must be positive")
        if not self.classes:
            raise TraceError("at least one request class is required")
        total = sum(c.weight for c in self.classes)
        if abs(total - 1.0) > 1e-9:
            raise TraceError(f"class weights must sum to 1.0, got {total}")
        for c in self.classes:
            if c.weight <= 0:
                raise TraceError("class weights must be positive")
            if c.shared_blocks < 0 or c.suffix_blocks[0] < 0:
                raise TraceError("block counts must be non-negative")
            if c.shared_blocks + c.suffix_blocks[0] < 1:
                raise TraceError("each request needs at least one block")
            if c.suffix_blocks[0] > c.suffix_blocks[1]:
                raise TraceError("suffix_blocks range is inverted")
            if c.output_tokens[0] < 1 or c.output_tokens[0] > c.output_tokens[1]:
                raise TraceError("output_tokens range must be >= 1 and ordered")


def class_key(prefix_blocks: Sequence[int], key_blocks: int = 2) -> int:
    """Class identity from the leading blocks (reference detector.py:41-45)."""
    if len(prefix_blocks) == 0:
        raise ValueError("class_key needs at least one block")
    return stable_key(CLASS_SALT, *[int(b) for b in prefix_blocks[:key_blocks]])


# -- packed (CSR) trace: what crosses the C-ABI ------------------------------------


@dataclass
class PackedTrace:
    """Structure-of-arrays trace. ``blocks[blk_off[i]:blk_off[i+1]]`` are
    request i's block hashes. ``arrival_us`` is ``round(arrival_s * 1e6)``
    with Python's half-even rounding (reference cluster.py:207)."""

    request_id: np.ndarray  # u64[R]
    arrival_s: np.ndarray  # f64[R]
    in_tokens: np.ndarray  # i64[R]
    out_tokens: np.ndarray  # i64[R]
    class_key: np.ndarray  # u64[R]
    blk_off: np.ndarray  # i64[R+1]
    blocks: np.ndarray  # u64[sum B]

    def __post_init__(self) -> None:
        self.arrival_us = np.rint(self.arrival_s * 1e6).astype(np.int64)

    def __len__(self) -> int:
        return int(self.request_id.shape[0])

    @property
    def n_blocks(self) -> np.ndarray:
        return np.diff(self.blk_off)

    def slice(self, n: int) -> "PackedTrace":
        """The first ``n`` records (decision k depends only on records[:k+1])."""
        off = self.blk_off[: n + 1]
        return PackedTrace(self.request_id[:n], self.arrival_s[:n], self.in_tokens[:n],
                           self.out_tokens[:n], self.class_key[:n], off.copy(),
                           self.blocks[: int(off[-1])])

    def record(self, i: int) -> TraceRecord:
        a, b = int(self.blk_off[i]), int(self.blk_off[i + 1])
        return TraceRecord(int(self.request_id[i]), float(self.arrival_s[i]),
                           tuple(int(x) for x in self.blocks[a:b].tolist()),
                           int(self.in_tokens[i]), int(self.out_tokens[i]),
                           int(self.class_key[i]))

    def records(self) -> list[TraceRecord]:
        return [self.record(i) for i in range(len(self))]

    @staticmethod
    def from_records(records: Sequence[TraceRecord]) -> "PackedTrace":
        if isinstance(records, PackedTrace):
            return records
        n = len(records)
        lens = np.fromiter((len(r.prefix_blocks) for r in records), dtype=np.int64, count=n)
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        blocks = np.fromiter((b & MASK64 for r in records for b in r.prefix_blocks),
                             dtype=np.uint64, count=int(off[-1]))
        return PackedTrace(
            np.fromiter((r.request_id & MASK64 for r in records), dtype=np.uint64, count=n),
            np.fromiter((r.arrival_s for r in records), dtype=np.float64, count=n),
            np.fromiter((r.input_tokens for r in records), dtype=np.int64, count=n),
            np.fromiter((r.output_tokens for r in records), dtype=np.int64, count=n),
            np.fromiter((r.class_key & MASK64 for r in records), dtype=np.uint64, count=n),
            off, blocks)


def concat_packed(parts: Sequence[PackedTrace]) -> PackedTrace:
    offs, base = [np.zeros(1, np.int64)], 0
    for p in parts:
        offs.append(p.blk_off[1:] + base)
        base += int(p.blk_off[-1])
    return PackedTrace(*(np.concatenate([getattr(p, f) for p in parts]) for f in
                         ("request_id", "arrival_s", "in_tokens", "out_tokens", "class_key")),
                       np.concatenate(offs), np.concatenate([p.blocks for p in parts]))


# -- file I/O ----------------------------------------------------------------------

_REQUIRED = ("id", "arrival_s", "blocks", "in", "out")


def _parse(text: str, line_no: int) -> TraceRecord:
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as exc:
        raise TraceError(f"invalid JSON: {exc.msg}", line_no) from exc
    if not isinstance(obj, dict):
        raise TraceError("record is not an object", line_no)
    missing = [f for f in _REQUIRED if f not in obj]
    if missing:
        raise TraceError(f"missing field {missing[0]!r}", line_no)
    rid, arrival, blocks, n_in, n_out = (obj[f] for f in _REQUIRED)
    if not isinstance(rid, int) or rid < 0:
        raise TraceError("id must be a non-negative integer", line_no)
    if isinstance(arrival, bool) or not isinstance(arrival, (int, float)) or arrival < 0:
        raise TraceError("arrival_s must be a non-negative number", line_no)
    if not isinstance(blocks, list) or not blocks:
        raise TraceError("blocks must be a non-empty list", line_no)
    if any(not isinstance(b, int) or b < 0 or b > MASK64 for b in blocks):
        raise TraceError("block hashes must be u64", line_no)
    if not isinstance(n_in, int) or n_in < 1:
        raise TraceError("in must be a positive integer", line_no)
    if not isinstance(n_out, int) or n_out < 1:
        raise TraceError("out must be a positive integer", line_no)
    cls = obj.get("class")
    if cls is None:
        cls = class_key(blocks)
    elif not isinstance(cls, int) or cls < 0 or cls > MASK64:
        raise TraceError("class must be u64", line_no)
    return TraceRecord(rid, float(arrival), tuple(blocks), n_in, n_out, cls)


def load_trace(path: str | Path) -> list[TraceRecord]:
    try:
        text = Path(path).read_text(encoding="utf-8")
    except OSError as exc:
        raise TraceError(f"cannot read trace file {path}: {exc}") from exc
    out: list[TraceRecord] = []
    last = -math.inf
    for no, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        rec = _parse(line, no)
        if rec.arrival_s < last:
            raise TraceError(f"arrival {rec.arrival_s} before previous {last}", no)
        last = rec.arrival_s
        out.append(rec)
    return out


_IO_LIB = None


def _io_lib():
    """librsimio.so (csrc/rsim_io.cpp, include/rsim_io.h), built in-tree by build()."""
    global _IO_LIB
    if _IO_LIB is None:
        import ctypes as C
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librsimio.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(path)
        P = C.c_void_p
        L.rsim_trace_parse_jsonl.argtypes = [C.c_char_p, C.c_int64, C.POINTER(P)]
        L.rsim_trace_parse_jsonl.restype = C.c_int
        L.rsim_trace_parse_count.argtypes = [P, C.POINTER(C.c_int64)]
        L.rsim_trace_parse_count.restype = C.c_int64
        L.rsim_trace_parse_copy.argtypes = [P] * 8
        L.rsim_trace_parse_copy.restype = None
        L.rsim_trace_parse_error.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.rsim_trace_parse_error.restype = C.c_char_p
        L.rsim_trace_parse_free.argtypes = [P]
        L.rsim_trace_parse_free.restype = None
        _IO_LIB = L
    return _IO_LIB


def load_trace_packed(path: str | Path) -> PackedTrace:
    """load_trace (reference trace.py:151-167) straight into a PackedTrace: the whole file
    is parsed by librsimio's one-pass C++ JSONL reader (same acceptance rules, checks and
    TraceError texts as _parse_line, trace.py:111-148), no per-line Python objects."""
    import ctypes as C
    try:
        data = Path(path).read_bytes()
    except OSError as exc:
        raise TraceError(f"cannot read trace file {path}: {exc}") from exc
    data.decode("utf-8")                                  # read_text's UnicodeDecodeError, unchanged
    L = _io_lib()
    h = C.c_void_p()
    st = L.rsim_trace_parse_jsonl(data, len(data), C.byref(h))
    try:
        if st != 0:
            line, a, prev = C.c_int64(), C.c_double(), C.c_double()
            msg = L.rsim_trace_parse_error(h, C.byref(line), C.byref(a), C.byref(prev)).decode()
            if st == 3:
                msg = f"arrival {a.value} before previous {prev.value}"
            raise TraceError(msg, int(line.value))
        nb = C.c_int64()
        n = int(L.rsim_trace_parse_count(h, C.byref(nb)))
        cols = (np.empty(n, np.uint64), np.empty(n, np.float64), np.empty(n, np.int64), np.empty(n, np.int64),
                np.empty(n, np.uint64), np.empty(n + 1, np.int64), np.empty(int(nb.value), np.uint64))
        L.rsim_trace_parse_copy(h, *(c.ctypes.data_as(C.c_void_p) for c in cols))
        return PackedTrace(*cols)
    finally:
        L.rsim_trace_parse_free(h)


def save_packed(trace: PackedTrace, path: str | Path) -> None:
    """Binary SoA/CSR trace file (numpy .npz, uncompressed): the packed columns as loaded
    into HBM, so a 1M-request trace round-trips without any per-record work."""
    with open(path, "wb") as fh:
        np.savez(fh, format=np.array([1]), request_id=trace.request_id, arrival_s=trace.arrival_s,
                 in_tokens=trace.in_tokens, out_tokens=trace.out_tokens, class_key=trace.class_key,
                 blk_off=trace.blk_off, blocks=trace.blocks)


def load_packed(path: str | Path) -> PackedTrace:
    """Inverse of save_packed; checks the CSR shape and arrival order like load_trace."""
    try:
        z = np.load(path, allow_pickle=False)
    except (OSError, ValueError) as exc:
        raise TraceError(f"cannot read trace file {path}: {exc}") from exc
    t = PackedTrace(*(z[f] for f in ("request_id", "arrival_s", "in_tokens", "out_tokens", "class_key",
                                     "blk_off", "blocks")))
    n = len(t)
    if t.blk_off.shape != (n + 1,) or t.blk_off[0] != 0 or int(t.blk_off[-1]) != t.blocks.shape[0] \
            or np.any(np.diff(t.blk_off) < 1):
        raise TraceError("packed trace: inconsistent CSR offsets")
    bad = np.nonzero(t.arrival_s[1:] < t.arrival_s[:-1])[0]
    if bad.size:
        i = int(bad[0]) + 1
        raise TraceError(f"arrival {float(t.arrival_s[i])} before previous {float(t.arrival_s[i - 1])}", i + 1)
    return t


def save_trace(records: Iterable[TraceRecord], path: str | Path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for r in records:
            fh.write(json.dumps({"id": r.request_id, "arrival_s": r.arrival_s,
                                 "blocks": list(r.prefix_blocks), "in": r.input_tokens,
                                 "out": r.output_tokens, "class": r.class_key},
                                separators=(",", ":")))
            fh.write("\n")


def observed_rate_rps(records: Sequence[TraceRecord]) -> float:
    if len(records) < 2:
        raise TraceError("need at least 2 records to measure a rate")
    span = records[-1].arrival_s - records[0].arrival_s
    if span <= 0:
        raise TraceError("trace spans zero time; rate is undefined")
    return (len(records) - 1) / span


def scale_trace(records: Sequence[TraceRecord], target_rate_rps: float) -> list[TraceRecord]:
    if target_rate_rps <= 0:
        raise TraceError("target rate must be positive")
    factor = observed_rate_rps(records) / target_rate_rps
    t0 = records[0].arrival_s
    return [dataclasses.replace(r, arrival_s=(r.arrival_s - t0) * factor) for r in records]


def scale_packed(trace: "PackedTrace", target_rate_rps: float) -> "PackedTrace":
    """scale_trace (reference trace.py) on a packed trace: arrival_s' = (arrival_s - t0) * factor
    with factor = observed rate / target, elementwise in IEEE doubles exactly as the
    per-record Python arithmetic; arrival_us is re-rounded half-even."""
    if target_rate_rps <= 0:
        raise TraceError("target rate must be positive")
    n = len(trace)
    if n < 2:
        raise TraceError("need at least 2 records to measure a rate")
    span = float(trace.arrival_s[-1]) - float(trace.arrival_s[0])
    if span <= 0:
        raise TraceError("trace spans zero time; rate is undefined")
    factor = ((n - 1) / span) / target_rate_rps
    arr = (trace.arrival_s - trace.arrival_s[0]) * factor
    return dataclasses.replace(trace, arrival_s=arr)


def validate_against_block_size(trace: PackedTrace, block_size: int) -> None:
    """ceil(in / block_size) must equal the block count (reference trace.py:271-281)."""
    want = -(-trace.in_tokens // block_size)
    bad = np.nonzero(want != trace.n_blocks)[0]
    if bad.size:
        i = int(bad[0])
        raise TraceError(
            f"record {int(trace.request_id[i])}: {int(trace.n_blocks[i])} blocks but "
            f"{int(trace.in_tokens[i])} tokens implies {int(want[i])} at block size {block_size}")


# -- synthetic generation --------------------------------------------------------------


def generate_synthetic_packed(spec: SyntheticSpec) -> PackedTrace:
    """Same trace as the reference generator, built as a PackedTrace.

    Arrival times and per-request sizes come from the same ``random.Random``
    streams in the same draw order; block hashes are ``stable_key`` values
    computed in bulk with numpy.
    """
    spec.validate()
    seed = spec.seed & MASK64
    times, cls_ids, seqs = [], [], []
    for ci, cls in enumerate(spec.classes):
        rng = random.Random(stable_key(seed, CLASS_RNG_SALT, ci))
        rate = cls.weight * spec.mean_rate_rps
        t = rng.expovariate(rate)
        k = 0
        while t < spec.duration_s:
            times.append(t)
            k += 1
            t += rng.expovariate(rate)
        cls_ids.append(np.full(k, ci, dtype=np.int64))
        seqs.append(np.arange(k, dtype=np.int64))
    t_arr = np.asarray(times, dtype=np.float64)
    ci_arr = np.concatenate(cls_ids) if cls_ids else np.zeros(0, np.int64)
    seq_arr = np.concatenate(seqs) if seqs else np.zeros(0, np.int64)
    order = np.lexsort((seq_arr, ci_arr, t_arr))  # tuple sort of (t, ci, seq)
    t_arr, ci_arr, seq_arr = t_arr[order], ci_arr[order], seq_arr[order]
    n = t_arr.shape[0]

    # per-class size draws, in arrival order within the class (= seq order)
    n_suffix = np.empty(n, dtype=np.int64)
    n_out = np.empty(n, dtype=np.int64)
    for ci, cls in enumerate(spec.classes):
        rng = random.Random(stable_key(seed, CLASS_RNG_SALT, ci, 1))
        idx = np.nonzero(ci_arr == ci)[0]  # already ascending in seq
        lo_s, hi_s = cls.suffix_blocks
        lo_o, hi_o = cls.output_tokens
        ri = rng.randint
        draws = [(ri(lo_s, hi_s), ri(lo_o, hi_o)) for _ in range(idx.shape[0])]
        if draws:
            d = np.asarray(draws, dtype=np.int64)
            n_suffix[idx], n_out[idx] = d[:, 0], d[:, 1]

    shared_n = np.asarray([c.shared_blocks for c in spec.classes], dtype=np.int64)
    shared = [stable_key_np(seed, SHARED_SALT, ci, np.arange(c.shared_blocks, dtype=np.uint64))
              for ci, c in enumerate(spec.classes)]
    lens = shared_n[ci_arr] + n_suffix
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    blocks = np.empty(int(off[-1]), dtype=np.uint64)
    # shared prefixes
    for ci in range(len(spec.classes)):
        sn = int(shared_n[ci])
        if sn == 0:
            continue
        rows = np.nonzero(ci_arr == ci)[0]
        pos = off[rows][:, None] + np.arange(sn)[None, :]
        blocks[pos.ravel()] = np.tile(shared[ci], rows.shape[0])
    # fresh suffixes: stable_key(seed, SUFFIX_SALT, ci, seq, pos)
    tot = int(n_suffix.sum())
    if tot:
        req = np.repeat(np.arange(n), n_suffix)
        start = np.repeat(np.cumsum(n_suffix) - n_suffix, n_suffix)
        pos = np.arange(tot) - start
        blocks[off[req] + shared_n[ci_arr[req]] + pos] = stable_key_np(
            seed, SUFFIX_SALT, ci_arr[req].astype(np.uint64), seq_arr[req].astype(np.uint64),
            pos.astype(np.uint64))
    # class_key = stable_key(CLASS_SALT, b0[, b1])
    first = blocks[off[:-1]] if n else np.zeros(0, np.uint64)
    two = lens >= 2
    ck = stable_key_np(CLASS_SALT, first)
    if n and two.any():
        second = blocks[off[:-1][two] + 1]
        ck = np.asarray(ck).copy()
        ck[two] = stable_key_np(CLASS_SALT, first[two], second)
    return PackedTrace(np.arange(n, dtype=np.uint64), t_arr, lens * spec.block_size, n_out,
                       np.asarray(ck, dtype=np.uint64).reshape(n), off, blocks)


def generate_synthetic_device(spec: SyntheticSpec, device: int = 0) -> PackedTrace:
    """generate_synthetic on the GPU (librsim rsim_synth_generate, csrc/rsim_synth.cuh):
    the same trace as generate_synthetic_packed, bit for bit, in milliseconds instead of
    seconds at 1M requests. Raises TraceError for an invalid spec, like the reference."""
    spec.validate()
    from . import _native
    rid, t, inp, out, ck, off, blocks = _native.synth_generate(spec, device)
    return PackedTrace(rid, t, inp, out, ck, off, blocks)


def generate_synthetic(spec: SyntheticSpec) -> list[TraceRecord]:
    return generate_synthetic_packed(spec).records()
