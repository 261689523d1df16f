"""Trace codec: librsimio's C++ JSONL reader (load_trace_packed) against the reference's
load_trace (trace.py:108-167) on the golden corpus tools/make_trace_golden.py recorded
from the reference itself -- records, or the exact TraceError text and line -- plus
round trips of generated traces through the JSONL and binary (.npz) formats."""
import json
import math
import os

import numpy as np
import pytest

import golden_cases as G
from paper_2603_15202_b200 import workloads as W
from paper_2603_15202_b200.trace import (PackedTrace, TraceError, load_packed, load_trace, load_trace_packed,
                                         save_packed, save_trace)

CASES = json.load(open(os.path.join(G.GOLDEN, "jsonl_cases.json")))


def _write(tmp_path, name, text):
    p = tmp_path / (name + ".jsonl")
    with open(p, "w", encoding="utf-8", newline="") as fh:
        fh.write(text)
    return p


def _same_float(a: float, b: str) -> bool:
    return repr(float(a)) == b or (math.isnan(a) and b == "nan")


@pytest.mark.parametrize("name", sorted(CASES))
def test_jsonl_reader_matches_reference(tmp_path, name):
    case = CASES[name]
    p = _write(tmp_path, name, case["text"])
    if "error" in case:
        with pytest.raises(TraceError) as ei:
            load_trace_packed(p)
        assert str(ei.value) == case["error"] and ei.value.line == case["line"]
        return
    t = load_trace_packed(p)
    want = case["records"]
    assert len(t) == len(want)
    for i, (rid, arr, blocks, n_in, n_out, cls) in enumerate(want):
        assert int(t.request_id[i]) == rid
        assert _same_float(float(t.arrival_s[i]), arr)
        assert t.blocks[t.blk_off[i]:t.blk_off[i + 1]].tolist() == blocks
        assert (int(t.in_tokens[i]), int(t.out_tokens[i]), int(t.class_key[i])) == (n_in, n_out, cls)


@pytest.mark.parametrize("name", sorted(CASES))
def test_python_mirror_matches_reference(tmp_path, name):
    """The pure-Python load_trace mirror agrees with the same corpus."""
    case = CASES[name]
    p = _write(tmp_path, name, case["text"])
    if "error" in case:
        with pytest.raises(TraceError) as ei:
            load_trace(p)
        assert str(ei.value) == case["error"]
        return
    got = [[int(r.request_id), r.arrival_s, list(r.prefix_blocks), r.input_tokens, r.output_tokens, r.class_key]
           for r in load_trace(p)]
    assert len(got) == len(case["records"])
    for g, w in zip(got, case["records"]):
        assert _same_float(g[1], w[1]) and [g[0]] + g[2:] == [w[0]] + w[2:]


def test_unsupported_ids_fail_loudly(tmp_path):
    p = _write(tmp_path, "bigid", '{"id":18446744073709551616,"arrival_s":0,"blocks":[1],"in":1,"out":1}\n')
    with pytest.raises(TraceError, match="64 bits"):
        load_trace_packed(p)


def test_missing_file(tmp_path):
    with pytest.raises(TraceError, match="cannot read trace file"):
        load_trace_packed(tmp_path / "nope.jsonl")


def _same(a: PackedTrace, b: PackedTrace):
    for f in ("request_id", "arrival_s", "in_tokens", "out_tokens", "class_key", "blk_off", "blocks", "arrival_us"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("maker", ["chat", "api", "agent"])
def test_round_trips(tmp_path, maker):
    t = {"chat": lambda: W.config1_chatbot()[0].slice(3000), "api": lambda: W.config2_api()[0].slice(2000),
         "agent": lambda: W.config3_agent(200)[0]}[maker]()
    p = tmp_path / "t.jsonl"
    save_trace(t.records(), p)
    _same(load_trace_packed(p), t)
    _same(PackedTrace.from_records(load_trace(p)), t)
    q = tmp_path / "t.npz"
    save_packed(t, q)
    _same(load_packed(q), t)


def test_binary_checks_order(tmp_path):
    t = W.config1_chatbot()[0].slice(10)
    t.arrival_s[5] = 0.0
    q = tmp_path / "bad.npz"
    save_packed(t, q)
    with pytest.raises(TraceError, match="before previous"):
        load_packed(q)
