"""bench.py end to end: the JSON line's contract keys, the decision-by-decision parity
check against the oracle, and the multi-GPU path (``--gpus 2`` self-launches two ranks
under torch.distributed.run; on a one-GPU box both ranks share the device and exchange
their per-decision partials through CUDA-IPC-mapped mailboxes)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(*args, timeout=900):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    return json.loads(lines[0])


def _expected_digest(workload, n):
    sys.path.insert(0, ROOT)
    import bench
    from paper_2603_15202_b200.cluster import run
    trace, cfg = bench.build_workload(workload)
    trace = trace.slice(n)
    return bench.chosen_digest(run(trace, cfg).chosen), len(trace)


def test_bench_single_gpu_line_has_parity():
    line = _bench("--workload", "chat16", "--extra", "", "--steps", "2", "--warmup", "3", "--whatif", "2000",
                  "--no-cpu")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "roofline", "e2e", "gpu_launches", "clocks", "parity", "decisions_sha256_16"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 2
    assert line["parity"]["mismatches"] == 0
    assert line["parity"]["decisions"] == line["config"]["requests"]
    assert line["gpu_launches"] > 0
    dig, _ = _expected_digest("chat16", line["config"]["requests"])
    assert line["decisions_sha256_16"] == dig


def test_bench_two_ranks_sharded():
    n = 150
    line = _bench("--gpus", "2", "--workload", "chat16", "--requests", str(n), "--steps", "1", "--warmup", "3",
                  "--whatif", "0", "--no-cpu")
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["requests"] == n
    assert line["parity"]["mismatches"] == 0 and line["parity"]["decisions"] == n
    assert len(line["ranks"]) == 2
    for r, ev in enumerate(line["ranks"]):
        assert ev["rank"] == r and ev["ipc_mailboxes_opened"] == 1
    assert line["ranks"][0]["shard"] == [0, 8] and line["ranks"][1]["shard"] == [8, 16]
    assert line["decision_latency_us"]["p50"] is not None
    dig, _ = _expected_digest("chat16", n)
    assert line["decisions_sha256_16"] == dig          # G = 2 makes exactly the G = 1 decisions
