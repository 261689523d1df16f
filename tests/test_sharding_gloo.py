"""The multi-GPU winner exchange, run as a world-size-2 gloo group on CPU:
every rank scores its contiguous shard, all-gathers the (min bits, tie count)
partials, and must reach the same decision as the reference argmin with
rotating tie-break over all instances (policies.py:92-101, 160-165)."""
import os
import random

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_15202_b200.sharding import (Partial, global_winner, local_partial, score_bits,
                                            shard_bounds)


def reference_argmin(scores, counter):
    best = min(scores)
    tied = [i for i, s in enumerate(scores) if s == best]
    if len(tied) == 1:
        return tied[0], counter
    return tied[counter % len(tied)], counter + 1


def _worker(rank, world, port, n_decisions, n_instances, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = random.Random(1234)                   # identical stream on every rank
    counter = 0x46B73E79F0C37C00                # stable_key(0, 0), cluster.py:90-94
    lo, hi = shard_bounds(n_instances, world, rank)
    picks = []
    for _ in range(n_decisions):
        scores = [float(rng.choice([1, 2, 3, 500, 1e300])) * rng.choice([1, 1, 2]) for _ in range(n_instances)]
        part, tied = local_partial(scores[lo:hi])
        gathered = [None] * world
        dist.all_gather_object(gathered, (part.min_bits, part.tie_count))
        owner, idx, counter = global_winner([Partial(*g) for g in gathered], counter)
        flag = [None] * world
        mine = lo + tied[idx] if owner == rank else None
        dist.all_gather_object(flag, mine)
        picks.append(flag[owner])
    if rank == 0:
        out.put(picks)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_instances", [7, 16, 33])
def test_two_rank_exchange_matches_reference_argmin(n_instances):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + n_instances
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 60, n_instances, q)) for r in range(2)]
    for p in procs:
        p.start()
    picks = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = random.Random(1234)
    counter = 0x46B73E79F0C37C00
    want = []
    for _ in range(60):
        scores = [float(rng.choice([1, 2, 3, 500, 1e300])) * rng.choice([1, 1, 2]) for _ in range(n_instances)]
        c, counter = reference_argmin(scores, counter)
        want.append(c)
    assert picks == want


def test_shard_bounds_cover_and_balance():
    for n in (1, 5, 64, 4096, 4097):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_score_bits_preserve_order():
    xs = [0.0, 1e-300, 0.5, 1.0, 1.0000000000000002, 500.0, 1e300, float("inf")]
    assert sorted(xs, key=score_bits) == xs
