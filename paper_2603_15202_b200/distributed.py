"""Sharded replay across GPUs.

Each rank owns a contiguous shard of the instances (``sharding.shard_bounds``)
in its own librsim handle; the whole trace and its chain keys are replicated.
Per decision every rank's replay kernel publishes one (min score bits, tie
count) partial into every peer's mailbox with a release store over NVLink
(peer-mapped device memory) and polls its own mailbox with acquire loads --
a device-initiated exchange, no host round trip and no NCCL call per
decision. The winner rule (``sharding.global_winner``) is evaluated
identically on every rank; only the owning rank commits, so per-request
outputs are merged across ranks afterwards (-1 where a rank did not own).

* ``run_sharded_local``: all ranks as handles of one process on one device
  (peers are plain device pointers) -- exercises the exchange protocol on a
  single GPU and is what the tests use.
* ``ShardedRouter``: one process per GPU under torchrun; mailbox IPC handles
  are exchanged once with ``torch.distributed.all_gather_object``.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _native
from .cluster import INT64_MAX, Sizing, native_config, sizing_for
from .config import ClusterConfig
from .trace import PackedTrace


def _merge(parts: list[np.ndarray]) -> np.ndarray:
    out = parts[0].copy()
    for p in parts[1:]:
        np.maximum(out, p, out=out)
    return out


def _load(h: _native.Handle, trace: PackedTrace):
    h.load(trace.arrival_us, trace.in_tokens, trace.out_tokens, trace.request_id, trace.blk_off, trace.blocks)


def run_sharded_local(trace: PackedTrace, config: ClusterConfig, world: int, *, device: int = 0,
                      ctas: int = 0, warps_per_cta: int = 0, repeats: int = 1) -> dict:
    """Replay ``trace`` with the instances split over ``world`` handles on one device."""
    sizing = sizing_for(trace, config)
    hs = [_native.Handle(native_config(config, sizing, device=device, world=world, rank=r, ctas=ctas,
                                       warps_per_cta=warps_per_cta)) for r in range(world)]
    try:
        ptrs = [h.mailbox() for h in hs]
        for h in hs:
            for r, p in enumerate(ptrs):
                h.set_peer(r, p)
            _load(h, trace)
        times = []
        for _ in range(repeats):
            errs = [None] * world
            ms = [0.0] * world

            def work(i):
                try:
                    ms[i] = hs[i].rerun()
                except Exception as exc:  # surfaced below
                    errs[i] = exc
            th = [threading.Thread(target=work, args=(i,)) for i in range(world)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            for e in errs:
                if e is not None:
                    raise e
            times.append(max(ms))
        n = len(trace)
        ch = _merge([h.decisions(0, n)[0] for h in hs])
        ht = _merge([h.decisions(0, n)[1] for h in hs])
        times3 = [h.request_times(0, n) for h in hs]
        return {"chosen": ch, "hit_tokens": ht,
                "first_sched_us": _merge([t[0] for t in times3]),
                "first_token_us": _merge([t[1] for t in times3]),
                "finish_us": _merge([t[2] for t in times3]),
                "device_ms": times}
    finally:
        for h in hs:
            h.close()


class ShardedRouter:
    """One rank of a sharded replay under torchrun (one process per GPU)."""

    def __init__(self, config: ClusterConfig, trace: PackedTrace, *, rank: int, world: int, device: int,
                 sizing: Sizing | None = None, comm_timeout_ms: int = 20000):
        import torch.distributed as dist
        self.trace = trace
        self.world, self.rank = world, rank
        sizing = sizing or sizing_for(trace, config)
        self.h = _native.Handle(native_config(config, sizing, device=device, world=world, rank=rank,
                                              comm_timeout_ms=comm_timeout_ms))
        handles = [None] * world
        dist.all_gather_object(handles, self.h.mailbox_ipc_handle())
        self.peers_opened = 0
        for r, hd in enumerate(handles):
            if r != rank:
                self.h.open_peer_ipc(r, hd)
                self.peers_opened += 1
        _load(self.h, trace)
        dist.barrier()

    def rerun(self) -> float:
        """Resident collective replay (all ranks call it); returns this rank's device ms."""
        return self.h.rerun()

    def local_decisions(self):
        return self.h.decisions(0, len(self.trace))

    def run_trace(self, trace: PackedTrace):
        """Collective end-to-end replay of host arrays: reset, H2D load, replay, drain, D2H of this
        rank's decisions, merged over ranks (each decision is committed by exactly one rank).
        Returns (chosen int32[n], hit_tokens int64[n]) on every rank."""
        import torch
        import torch.distributed as dist
        h = self.h
        h.reset()
        n = len(trace)
        _load(h, trace)
        h.replay(0, n)
        h.drain()
        ch, ht = h.decisions(0, n)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
        t = torch.from_numpy(np.stack([ch.astype(np.int64), ht.astype(np.int64)])).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = t.cpu().numpy()
        self.trace = trace
        return t[0].astype(np.int32), t[1]

    def close(self):
        self.h.close()
