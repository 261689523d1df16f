"""Instance sharding across GPUs and the per-decision winner exchange.

Instances are independent except through routing (reference cluster.py:8-11),
so GPU g owns a contiguous id range; every GPU probes and scores only its
own instances and contributes one partial per decision. The global winner
must equal the reference's ``_argmin`` + ``TieBreaker.pick`` over all
instances in ascending id order (policies.py:92-101, 160-165):

    best   = min over all scores
    tied   = ids with score == best, ascending
    chosen = tied[counter % len(tied)] if len(tied) > 1 (then counter += 1)

With contiguous shards, "ascending id" is rank-major, so the winner follows
from the rank-ordered partials ``(min score bits, tie count)`` alone: the
global tie count T is the sum of the counts of ranks whose minimum equals the
global minimum, kk = counter mod T locates the owning rank by prefix sums of
those counts, and the owner picks its local (kk - prefix)-th tied instance.
This is the same rule the replay kernel applies across the CTAs of a cluster
(csrc/rsim_kernels.cuh), one level up. These host functions define the rule
for the multi-GPU path and are exercised with a gloo world in the tests.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass


def shard_bounds(n_instances: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank ``rank`` (sizes differ by at most one)."""
    base, extra = divmod(n_instances, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def score_bits(x: float) -> int:
    """Order-preserving u64 image of a non-negative double (scores are >= 0)."""
    return struct.unpack("<Q", struct.pack("<d", float(x)))[0]


NO_CANDIDATE = (1 << 64) - 1


@dataclass(frozen=True)
class Partial:
    min_bits: int      # NO_CANDIDATE if the shard has no candidate
    tie_count: int


def local_partial(scores) -> tuple[Partial, list[int]]:
    """Partial of one shard plus its tied local indices (ascending)."""
    if len(scores) == 0:
        return Partial(NO_CANDIDATE, 0), []
    bits = [score_bits(s) for s in scores]
    m = min(bits)
    tied = [i for i, b in enumerate(bits) if b == m]
    return Partial(m, len(tied)), tied


def global_winner(partials: list[Partial], counter: int) -> tuple[int, int, int]:
    """(owner rank, index into that rank's tied list, new counter)."""
    gmin = min(p.min_bits for p in partials)
    counts = [p.tie_count if p.min_bits == gmin else 0 for p in partials]
    total = sum(counts)
    if total == 0:
        raise ValueError("no candidates on any rank")
    kk = 0
    if total > 1:
        kk = counter % total
        counter += 1
    prefix = 0
    for r, c in enumerate(counts):
        if kk < prefix + c:
            return r, kk - prefix, counter
        prefix += c
    raise AssertionError("unreachable")
