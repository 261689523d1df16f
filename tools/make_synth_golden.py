"""Golden fingerprints of the reference's synthetic generator (tests/golden/synth_golden.json).

Runs the reference's own ``routesim.trace.generate_synthetic`` (trace.py:218-268, imported
from /root/reference in this container) on the specs in SPECS and records, per spec, the
request count and a sha256 per PackedTrace column (request_id, arrival_s as f64 bits,
input_tokens, output_tokens, class_key, blk_off, blocks), plus the first rows in clear.
tests/test_synth.py checks the host generator (CPU) and the device generator
(rsim_synth_generate, GPU) against these; the reference never runs on the GPU box.

Usage: python tools/make_synth_golden.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from refcompat import import_reference  # noqa: E402

CHAT = "tuple((1 / 8, 8 + 4 * i, (2, 12), (16, 128)) for i in range(8))"
# name: (duration_s, mean_rate_rps, classes as (weight, shared, suffix, output) tuples, seed, block_size)
SPECS = {
    "chat_cfg1": f"(10000 / 48.0, 48.0, {CHAT}, 0, 16)",
    "api_cfg2": "(100000 / 384.0, 384.0, tuple((1 / 32, 64, (1, 4), (8, 64)) for _ in range(32)), 1, 16)",
    "chat1024": f"(100000 / 3072.0, 3072.0, {CHAT}, 0, 16)",
    "large_cfg4": f"(1000000 / 12288.0, 12288.0, {CHAT}, 0, 16)",
    "hotspot": "(3000 / 60.0, 60.0, ((0.6, 16, (1, 3), (16, 96)),) + tuple(((1 - 0.6) / 6, 8, (1, 4), (16, 64)) "
               "for _ in range(6)), 0, 16)",
    "one_class_fixed": "(50.0, 10.0, ((1.0, 0, (1, 1), (1, 1)),), 3, 16)",
    "rejection_ranges": "(200.0, 25.0, ((0.25, 0, (1, 5), (1, 1000)), (0.25, 3, (0, 4), (3, 3)), "
                        "(0.5, 1, (0, 0), (5, 9))), 11, 4)",
    "seed_2p32": "(100.0, 20.0, ((0.5, 2, (0, 3), (1, 9)), (0.5, 6, (1, 5), (1, 30))), 1 << 32, 16)",
    "seed_big": "(100.0, 20.0, ((0.5, 2, (0, 3), (1, 9)), (0.5, 6, (1, 5), (1, 30))), (1 << 64) - 12345, 16)",
    "seed_negative": "(100.0, 20.0, ((0.5, 2, (0, 3), (1, 9)), (0.5, 6, (1, 5), (1, 30))), -7, 16)",
    "many_classes": "(400.0, 30.0, tuple((1 / 40, i % 5, (0 if i % 5 else 1, 2 + i % 7), (1, 2 + i)) "
                    "for i in range(40)), 5, 8)",
    "sparse_short": "(0.5, 3.0, ((0.9, 4, (1, 2), (1, 4)), (0.1, 2, (1, 2), (1, 4))), 2, 16)",
}


def columns(records):
    n = len(records)
    lens = np.array([len(r.prefix_blocks) for r in records], dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    blocks = np.fromiter((b for r in records for b in r.prefix_blocks), dtype=np.uint64, count=int(off[-1]))
    return {
        "request_id": np.array([r.request_id for r in records], dtype=np.uint64),
        "arrival_s": np.array([r.arrival_s for r in records], dtype=np.float64),
        "in_tokens": np.array([r.input_tokens for r in records], dtype=np.int64),
        "out_tokens": np.array([r.output_tokens for r in records], dtype=np.int64),
        "class_key": np.array([r.class_key for r in records], dtype=np.uint64),
        "blk_off": off,
        "blocks": blocks,
    }


def digest(cols):
    return {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in cols.items()}


def main():
    import_reference()
    from routesim.trace import ClassSpec, SyntheticSpec, generate_synthetic
    out = {"_source": "routesim.trace.generate_synthetic run in this container (tools/make_synth_golden.py)"}
    for name, expr in SPECS.items():
        dur, rate, classes, seed, bs = eval(expr)
        spec = SyntheticSpec(dur, rate, tuple(ClassSpec(*c) for c in classes), seed=seed, block_size=bs)
        t0 = time.time()
        recs = generate_synthetic(spec)
        cols = columns(recs)
        out[name] = {"spec": expr, "n": len(recs), "n_blocks": int(cols["blk_off"][-1]), "sha256": digest(cols),
                     "head": {k: [float(x) if k == "arrival_s" else int(x) for x in v[:4]] for k, v in cols.items()},
                     "reference_seconds": round(time.time() - t0, 2)}
        print(f"{name:18s} n={len(recs):8d} {time.time() - t0:6.1f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "synth_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
