"""Host-side 64-bit hashing (splitmix64 chain keys).

Scalar functions restate ``routesim.hashing`` (reference
``pkg/src/routesim/hashing.py:15-47``) for API parity; the ``*_np`` variants
are vectorised numpy versions used to build traces and seeds without Python
loops. The hot-path chain hashing runs on the GPU (``librsim`` kernel
``k1_chain_keys``); these helpers only feed it and check it.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN64 = 0x9E3779B97F4A7C15  # splitmix increment, also the chain seed (hashing.py:12)
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def splitmix64(value: int) -> int:
    """splitmix64 finaliser (hashing.py:15-20)."""
    z = (value + GOLDEN64) & MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def combine64(acc: int, value: int) -> int:
    """Fold ``value`` into ``acc`` (hashing.py:23-25)."""
    return splitmix64((acc ^ value) & MASK64)


def stable_key(*values: int) -> int:
    """Order-sensitive key of a tuple, folded from the chain seed (hashing.py:28-33)."""
    acc = GOLDEN64
    for v in values:
        acc = combine64(acc, v & MASK64)
    return acc


def chain_keys(blocks) -> list[int]:
    """Cumulative prefix-chain keys (hashing.py:36-47)."""
    out = []
    acc = GOLDEN64
    for b in blocks:
        acc = combine64(acc, b & MASK64)
        out.append(acc)
    return out


# -- numpy (uint64 arithmetic wraps mod 2**64) ----------------------------------

_U = np.uint64


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    z = np.asarray(x, dtype=_U) + _U(GOLDEN64)
    z = (z ^ (z >> _U(30))) * _U(_M1)
    z = (z ^ (z >> _U(27))) * _U(_M2)
    return z ^ (z >> _U(31))


def combine64_np(acc, value) -> np.ndarray:
    return splitmix64_np(np.asarray(acc, dtype=_U) ^ np.asarray(value, dtype=_U))


def stable_key_np(*values) -> np.ndarray:
    """Vectorised ``stable_key``: each argument is a scalar or a broadcastable array."""
    with np.errstate(over="ignore"):
        acc = np.asarray(_U(GOLDEN64))
        for v in values:
            if isinstance(v, (int, np.integer)):
                v = _U(int(v) & MASK64)
            acc = combine64_np(acc, np.asarray(v).astype(_U, copy=False))
        return acc


def chain_keys_np(blocks: np.ndarray) -> np.ndarray:
    """Chain keys of one block sequence (sequential by construction)."""
    out = np.empty(len(blocks), dtype=_U)
    acc = GOLDEN64
    for i, b in enumerate(blocks.tolist()):
        acc = combine64(acc, b)
        out[i] = acc
    return out
