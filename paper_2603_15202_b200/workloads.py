"""The five benchmark/parity workloads of BASELINE.json.

Each builder returns ``(PackedTrace, ClusterConfig)``. Configs 1, 2 and 4
use the reference's synthetic generator semantics (``generate_synthetic``,
reference trace.py:218-268); config 3 is a multi-turn coding-agent trace
built in the reference's trace schema (the reference has no multi-turn
generator); config 5 is a family of hand-built adversarial traces.
"""

from __future__ import annotations

import numpy as np

from .config import CacheConfig, ClusterConfig, CostModel, PolicyConfig
from .hashing import MASK64, stable_key_np
from .trace import (CLASS_SALT, ClassSpec, PackedTrace, SyntheticSpec, concat_packed,
                    generate_synthetic_packed)

OUTPUT_SALT = 0x0F_0C0DE  # reference engine.py:34
_generate = generate_synthetic_packed


def use_device_generator(device: int = 0) -> None:
    """Build the synthetic workloads with the GPU generator (trace.generate_synthetic_device,
    bit-identical to the host one) -- bench.py's setup; tests keep the host generator."""
    global _generate
    from .trace import generate_synthetic_device
    _generate = lambda spec: generate_synthetic_device(spec, device)  # noqa: E731
CHAT_CLASSES = tuple(ClassSpec(1 / 8, 8 + 4 * i, (2, 12), (16, 128)) for i in range(8))


def chat_spec(n_requests: float, rate_rps: float, seed: int = 0) -> SyntheticSpec:
    return SyntheticSpec(duration_s=n_requests / rate_rps, mean_rate_rps=rate_rps,
                         classes=CHAT_CLASSES, seed=seed)


def config1_chatbot(seed: int = 0):
    """16 instances, ~10k requests at 48 req/s (SURVEY cfg 1)."""
    trace = _generate(chat_spec(10000, 48.0, seed))
    return trace, ClusterConfig(n_instances=16, cache=CacheConfig(16, 40000), seed=0)


def config2_api(n_requests: int = 100_000, seed: int = 1):
    """64 instances, ~100k requests sharing 32 1024-token system prompts (SURVEY cfg 2)."""
    spec = SyntheticSpec(duration_s=n_requests / 384.0, mean_rate_rps=384.0,
                         classes=tuple(ClassSpec(1 / 32, 64, (1, 4), (8, 64)) for _ in range(32)),
                         seed=seed)
    return _generate(spec), ClusterConfig(n_instances=64,
                                                          cache=CacheConfig(16, 40000), seed=0)


def chat_cluster(n_instances: int, n_requests: int, per_instance_rps: float = 3.0, seed: int = 0):
    """Chat class mix at ``per_instance_rps`` per instance (SURVEY cfg 4 / 1024-instance target)."""
    rate = per_instance_rps * n_instances
    trace = _generate(chat_spec(n_requests, rate, seed))
    return trace, ClusterConfig(n_instances=n_instances, cache=CacheConfig(16, 40000), seed=0)


def hotspot(n_instances: int = 16, n_requests: int = 3000, hot_fraction: float = 0.6, rate_rps: float = 60.0,
            n_cold: int = 6, seed: int = 0):
    """One hot system prompt taking ``hot_fraction`` of arrivals next to ``n_cold``
    cold classes: the prefix-hotspot regime the reference detector watches
    (detector.py:1-23)."""
    cold = (1.0 - hot_fraction) / n_cold
    classes = (ClassSpec(hot_fraction, 16, (1, 3), (16, 96)),) + tuple(
        ClassSpec(cold, 8, (1, 4), (16, 64)) for _ in range(n_cold))
    spec = SyntheticSpec(duration_s=n_requests / rate_rps, mean_rate_rps=rate_rps, classes=classes, seed=seed)
    return _generate(spec), ClusterConfig(n_instances=n_instances, cache=CacheConfig(16, 40000),
                                                          seed=seed)


def hotspot_detector(n_instances: int = 64, n_requests: int = 20_000, window_s: float = 5.0, seed: int = 0):
    """``hotspot`` at 2.5 req/s per instance with the reference detector on (detector.py)."""
    import dataclasses
    from .config import DetectorConfig
    trace, cfg = hotspot(n_instances, n_requests, 0.6, 2.5 * n_instances, seed=seed)
    return trace, dataclasses.replace(cfg, detector=DetectorConfig(window_s=window_s))


def config4_large(n_requests: int = 1_000_000, seed: int = 0):
    """4096 instances, ~1M requests at 3 req/s/instance (SURVEY cfg 4)."""
    return chat_cluster(4096, n_requests, 3.0, seed)


def config3_agent(n_requests: int = 20_000, n_instances: int = 256, capacity: int = 16_384,
                  seed: int = 3, block_size: int = 16, rate_per_instance: float = 0.5,
                  max_blocks: int = 2048):
    """Multi-turn coding-agent sessions with deep prefix reuse (SURVEY cfg 3).

    Sessions share a 256-block repo prompt. Turn k+1's blocks are turn k's
    blocks, then turn k's output-block hashes ``stable_key(0x0F0C0DE, rid, idx)``
    (the keys the engine inserts at finish, reference engine.py:363-372, so the
    next turn fully hits the previous chain on the instance that served it),
    then 16-128 fresh blocks. A session ends when the next turn would exceed
    ``max_blocks`` (32k tokens at 16-token blocks) or after its drawn turn count.
    Think time between turns (20-60 s) exceeds the service time.
    """
    rng = np.random.default_rng(seed)
    rate = rate_per_instance * n_instances
    repo = stable_key_np(seed, 0xA9E7_0001, np.arange(256, dtype=np.uint64))
    # generate sessions until enough turns exist, then keep the earliest n_requests arrivals
    turns = []  # (arrival_s, session, turn, blocks(list of arrays), out)
    t_session = 0.0
    session = 0
    horizon = n_requests / rate
    while True:
        t_session += rng.exponential(1.0 / (rate / 12.0))
        if t_session > horizon and len(turns) >= n_requests:
            break
        n_turns = int(rng.integers(4, 40))
        ctx = [repo]
        ctx_len = 256
        t = t_session
        prev = None
        for k in range(n_turns):
            if prev is not None:
                nob = -(-prev[1] // block_size)
                ctx.append(("out", prev[0], nob))
                ctx_len += nob
            n_new = int(rng.integers(16, 129))
            if ctx_len + n_new > max_blocks:
                break
            fresh = stable_key_np(seed, 0xA9E7_0002, np.uint64(session), np.uint64(k),
                                  np.arange(n_new, dtype=np.uint64))
            ctx.append(fresh)
            ctx_len += n_new
            out = int(rng.integers(64, 513))
            turns.append((t, session, k, list(ctx), out))
            prev = (len(turns) - 1, out)
            t += float(rng.uniform(20.0, 60.0))
        session += 1
        if session > 10 * n_requests:
            break
    # order by arrival; request ids are positions in that order
    order = sorted(range(len(turns)), key=lambda i: (turns[i][0], turns[i][1], turns[i][2]))[:n_requests]
    new_id = {old: new for new, old in enumerate(order)}
    lens, blocks_parts, arr, outs = [], [], [], []
    for old in order:
        t, _s, _k, ctx, out = turns[old]
        parts = []
        for piece in ctx:
            if isinstance(piece, tuple):
                _, rid_prev_old, nob = piece
                rid_prev = new_id[rid_prev_old]  # earlier turn, so inside the arrival-order prefix
                parts.append(stable_key_np(OUTPUT_SALT, np.uint64(rid_prev),
                                           np.arange(nob, dtype=np.uint64)))
            else:
                parts.append(piece)
        b = np.concatenate(parts).astype(np.uint64)
        blocks_parts.append(b)
        lens.append(b.shape[0])
        arr.append(t)
        outs.append(out)
    n = len(order)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.asarray(lens, dtype=np.int64), out=off[1:])
    blocks = np.concatenate(blocks_parts) if blocks_parts else np.zeros(0, np.uint64)
    first = blocks[off[:-1]]
    second = blocks[off[:-1] + 1]
    trace = PackedTrace(np.arange(n, dtype=np.uint64), np.asarray(arr, dtype=np.float64),
                        np.asarray(lens, dtype=np.int64) * block_size,
                        np.asarray(outs, dtype=np.int64),
                        np.asarray(stable_key_np(CLASS_SALT, first, second), dtype=np.uint64),
                        off, blocks)
    cfg = ClusterConfig(n_instances=n_instances, cache=CacheConfig(block_size, capacity), seed=0)
    return trace, cfg


# -- config 5: adversarial traces ---------------------------------------------------------


def _records(rows, block_size=16):
    """rows: (arrival_s, blocks(list[int]), in_tokens, out_tokens)."""
    n = len(rows)
    lens = np.asarray([len(r[1]) for r in rows], dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    blocks = np.asarray([b & MASK64 for r in rows for b in r[1]], dtype=np.uint64)
    first = np.asarray([r[1][0] for r in rows], dtype=np.uint64)
    return PackedTrace(np.arange(n, dtype=np.uint64), np.asarray([r[0] for r in rows], np.float64),
                       np.asarray([r[2] for r in rows], np.int64), np.asarray([r[3] for r in rows], np.int64),
                       np.asarray(stable_key_np(CLASS_SALT, first), dtype=np.uint64).reshape(n), off, blocks)


def adversarial(case: str, n_instances: int = 16, seed: int = 0):
    """Hand-built traces stressing the multiplication-failure conditions.

    cases: ``same_time_ties`` (K identical requests at one timestamp onto an
    idle cluster: N-way ties, rotation), ``zero_bs`` (bs 0 vs 1 instances
    tie through the max(bs,1) floor), ``full_hits`` (full-cache hits,
    new_prefill floor 1), ``ragged`` (input not a multiple of the block
    size), ``out1`` (single-token outputs finish at first token),
    ``step_boundary`` (arrivals exactly at step-end times and equal
    timestamps), ``tight_capacity`` (eviction with equal (touch, depth)
    siblings), ``mixed`` (all of the above interleaved, N not a multiple
    of 32).
    """
    rng = np.random.default_rng(seed)
    bs = 16
    rows = []
    if case == "same_time_ties":
        for k in range(4 * n_instances):
            rows.append((0.5, [7, 8, 9], 48, 4))
        for k in range(4 * n_instances):
            rows.append((1.0 + 0.25 * (k // n_instances), [100 + (k % 3), 200], 32, 2))
    elif case == "zero_bs":
        t = 0.0
        for k in range(6 * n_instances):
            rows.append((t, [int(rng.integers(1, 4)), 5000 + k], 32, int(rng.integers(1, 3))))
            t += 0.0125 * float(rng.integers(0, 3))
    elif case == "full_hits":
        t = 0.0
        for k in range(8 * n_instances):
            fam = int(rng.integers(0, 3))
            nb = 2 + fam
            rows.append((t, [9000 + 10 * fam + j for j in range(nb)], nb * bs - int(rng.integers(0, 2)) * 7,
                         int(rng.integers(1, 6))))
            t += 0.003 * float(rng.integers(0, 4))
    elif case == "ragged":
        t = 0.0
        for k in range(6 * n_instances):
            n_in = int(rng.integers(1, 200))
            nb = -(-n_in // bs)
            fam = int(rng.integers(0, 4))
            blocks = [777 + fam] + [int(x) for x in rng.integers(1, 1 << 62, size=nb - 1)]
            rows.append((t, blocks, n_in, int(rng.integers(1, 40))))
            t += float(rng.uniform(0.0, 0.01))
    elif case == "out1":
        t = 0.0
        for k in range(6 * n_instances):
            rows.append((t, [31, 32 + (k % 5)], 32, 1))
            t += 0.002
    elif case == "step_boundary":
        # default cost model: prefill of 32 tokens = 8.2 ms, decode of n seqs = 20+n ms;
        # arrivals land on multiples of those step ends and repeat timestamps
        t = 0.0
        for k in range(6 * n_instances):
            rows.append((round(t, 6), [41, 42, 43 + (k % 4)][: 1 + (k % 3)], 16 * (1 + (k % 3)), 2 + (k % 3)))
            if k % 3 == 2:
                t += [0.0082, 0.021, 0.0292, 0.022][k % 4]
    elif case == "tight_capacity":
        t = 0.0
        for k in range(10 * n_instances):
            fam = int(rng.integers(0, 6))
            nb = int(rng.integers(2, 7))
            blocks = [50 + fam, 60 + fam] + [int(x) for x in rng.integers(1, 1 << 62, size=nb - 2)]
            rows.append((t, blocks, nb * bs, int(rng.integers(1, 40))))
            t += float(rng.choice([0.0, 0.001, 0.02]))
    elif case == "mixed":
        parts = [adversarial(c, n_instances, seed)[0] for c in
                 ("same_time_ties", "zero_bs", "full_hits", "ragged", "out1", "step_boundary")]
        shift = 0.0
        shifted = []
        for p in parts:
            q = PackedTrace(p.request_id, p.arrival_s + shift, p.in_tokens, p.out_tokens, p.class_key,
                            p.blk_off, p.blocks)
            shifted.append(q)
            shift = float(q.arrival_s[-1]) + 0.0005
        tr = concat_packed(shifted)
        tr = PackedTrace(np.arange(len(tr), dtype=np.uint64), tr.arrival_s, tr.in_tokens, tr.out_tokens,
                         tr.class_key, tr.blk_off, tr.blocks)
        return tr, ClusterConfig(n_instances=n_instances, cache=CacheConfig(16, 64), seed=seed)
    else:
        raise ValueError(f"unknown adversarial case {case!r}")
    cap = 24 if case == "tight_capacity" else None
    cm = CostModel()
    return _records(rows), ClusterConfig(n_instances=n_instances, cost_model=cm,
                                         cache=CacheConfig(16, cap), seed=seed,
                                         policy=PolicyConfig())


ADVERSARIAL_CASES = ("same_time_ties", "zero_bs", "full_hits", "ragged", "out1", "step_boundary",
                     "tight_capacity", "mixed")


def adversarial_stream(n_instances: int = 64, n_requests: int = 100_000, capacity: int = 256, seed: int = 5):
    """BASELINE configs[4] at bench scale: the multiplication-failure conditions of
    ``adversarial`` interleaved over a long trace -- bursts of identical requests at one
    timestamp onto idle instances (N-way ties through the max(bs, 1) floor and the rotating
    tie-break), full-cache hits of a few short families (new_prefill floor 1), single-token
    outputs, ragged inputs, arrivals repeating timestamps, and a tight KV$ capacity whose
    evictions meet equal (touch, depth) siblings."""
    rng = np.random.default_rng(seed)
    bs = 16
    kind = rng.choice(4, size=n_requests, p=[0.3, 0.3, 0.15, 0.25])
    gaps = rng.choice([0.0, 0.0, 0.0005, 0.002, 0.0082, 0.021], size=n_requests)
    burst = kind == 0                      # bursts: the same timestamp as the previous request
    gaps[burst] = 0.0
    arrival = np.cumsum(gaps) * (64.0 / n_instances)
    rows = []
    for k in range(n_requests):
        c = int(kind[k])
        if c == 0:                         # identical requests: one of 4 tiny families
            fam = int(rng.integers(0, 4))
            rows.append((float(arrival[k]), [7 + fam, 8 + fam], 32, 2))
        elif c == 1:                       # full hits of short families, input 1 token short or exact
            fam = int(rng.integers(0, 6))
            nb = 2 + fam % 3
            rows.append((float(arrival[k]), [9000 + 10 * fam + j for j in range(nb)],
                         nb * bs - int(rng.integers(0, 2)) * 7, int(rng.integers(1, 6))))
        elif c == 2:                       # single-token outputs
            rows.append((float(arrival[k]), [31, 32 + k % 5], 32, 1))
        else:                              # ragged inputs over a shared first block
            n_in = int(rng.integers(1, 200))
            nb = -(-n_in // bs)
            blocks = [777 + int(rng.integers(0, 4))] + [int(x) for x in rng.integers(1, 1 << 62, size=nb - 1)]
            rows.append((float(arrival[k]), blocks, n_in, int(rng.integers(1, 40))))
    return _records(rows), ClusterConfig(n_instances=n_instances, cost_model=CostModel(),
                                         cache=CacheConfig(bs, capacity), seed=seed, policy=PolicyConfig())
