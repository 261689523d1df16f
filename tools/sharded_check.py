"""One rank of a torchrun sharded replay check (tests/test_device_sharded.py).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port P tools/sharded_check.py CASE N_REQUESTS

Every rank owns a contiguous instance shard in its own process; the mailbox
IPC handles travel over a gloo group (the ranks may share one GPU). The merged
decisions must equal the golden (reference) decisions of the case.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_cases as G  # noqa: E402
from paper_2603_15202_b200.distributed import ShardedRouter  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
ndev = torch.cuda.device_count()
dev = int(os.environ.get("LOCAL_RANK", rank)) % ndev
torch.cuda.set_device(dev)
trace, cfg = G.build(name)
trace = trace.slice(min(n, len(trace)))
want = G.expected(name)
r = ShardedRouter(cfg, trace, rank=rank, world=world, device=dev)
ch, ht = r.run_trace(trace)
ok = np.array_equal(ch, want["chosen"][:len(trace)]) and np.array_equal(ht, want["hit_tokens"][:len(trace)])
r.close()
if rank == 0:
    print(f"sharded {name} world={world} decisions={len(trace)}: {'OK' if ok else 'MISMATCH'}", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
