"""INTEGRATION.md's reference-side binding (routesim/gpu.py) is executed, not just shown:
its rsim_config mirror must match librsim's field for field (CPU), and its run_on_gpu must
reproduce the reference's decisions on golden traces (B200)."""
import ctypes
import os
import re
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# routesim/gpu\.py.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its routesim/gpu.py block"
    if "routesim.hashing" not in sys.modules:           # the reference is not importable on the GPU box
        from paper_2603_15202_b200 import hashing
        pkg = sys.modules.setdefault("routesim", types.ModuleType("routesim"))
        mod = types.ModuleType("routesim.hashing")
        mod.stable_key = hashing.stable_key
        pkg.hashing = mod
        sys.modules["routesim.hashing"] = mod
    os.environ["RSIM_LIBRARY"] = os.path.join(ROOT, "paper_2603_15202_b200", "librsim.so")
    ns = {"__name__": "routesim_gpu"}
    exec(compile(m.group(1), "INTEGRATION.md:routesim/gpu.py", "exec"), ns)
    return ns


def test_binding_struct_matches_library():
    from paper_2603_15202_b200 import _native
    ns = _binding()
    cfg = ns["_Cfg"]
    assert ctypes.sizeof(cfg) == _native.lib().rsim_config_size()
    ours = [(n, t) for n, t in _native.Config._fields_]
    theirs = [(n, t) for n, t in cfg._fields_]
    assert [n for n, _ in ours] == [n for n, _ in theirs]
    for (n, a), (_, b) in zip(ours, theirs):
        assert ctypes.sizeof(a) == ctypes.sizeof(b), n
        assert getattr(_native.Config, n).offset == getattr(cfg, n).offset, n


def test_binding_fills_every_policy():
    import golden_cases as G
    ns = _binding()
    for name in ("cfg1_chatbot_full", "policy_vllm", "policy_least_bs", "policy_linear_cap", "policy_filter",
                 "policy_simulate_mistuned", "stale_5ms"):
        if name not in G.names():
            continue
        trace, cfg = G.build(name)
        c = ns["make_config"](cfg, len(trace), 64)
        assert c.struct_size == ctypes.sizeof(ns["_Cfg"]) and c.abi_version == 2
        assert c.policy == {"multiplicative": 0, "vllm": 1, "least_bs": 2, "linear": 3, "filter": 4,
                            "simulate": 5}[cfg.policy.kind]


def test_truncated_struct_is_rejected():
    """A binding that stops early (round-1 INTEGRATION.md's _Cfg ended at expected_keys) is refused
    by rsim_create before any field past its end is read; no GPU needed for the check."""
    from paper_2603_15202_b200 import _native
    L = _native.lib()
    c = _native.Config()
    c.struct_size = 168
    h = ctypes.c_void_p()
    assert L.rsim_create(ctypes.byref(c), ctypes.byref(h)) == _native.E_INVALID
    assert b"layout mismatch" in L.rsim_last_error(None)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1_chatbot_full", "adv_tight_capacity", "policy_simulate_mistuned",
                                  "stale_50ms_n16", "adv_mixed_n33"])
def test_binding_reproduces_reference(name):
    import golden_cases as G
    ns = _binding()
    trace, cfg = G.build(name)
    want = G.expected(name)
    got = ns["run_on_gpu"](list(trace.records()), cfg)
    assert np.array_equal(np.array([c for c, _ in got]), want["chosen"])
    assert np.array_equal(np.array([h for _, h in got]), want["hit_tokens"])


@pytest.mark.gpu
def test_binding_generates_reference_trace():
    """The binding's generate_synthetic_on_gpu returns the reference generator's records
    (fingerprints in tests/golden/synth_golden.json)."""
    import hashlib
    import json
    from paper_2603_15202_b200.trace import ClassSpec, PackedTrace, SyntheticSpec, TraceRecord
    ns = _binding()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "synth_golden.json")))
    for name in ("chat_cfg1", "rejection_ranges", "seed_negative"):
        dur, rate, classes, seed, bs = eval(gold[name]["spec"])
        spec = SyntheticSpec(dur, rate, tuple(ClassSpec(*c) for c in classes), seed=seed, block_size=bs)
        recs = ns["generate_synthetic_on_gpu"](spec, record=TraceRecord)
        tr = PackedTrace.from_records(recs)
        assert len(recs) == gold[name]["n"]
        for col, want in gold[name]["sha256"].items():
            assert hashlib.sha256(np.ascontiguousarray(getattr(tr, col)).tobytes()).hexdigest() == want, (name, col)
