"""Host side of the device detector (no GPU): class tracks and config gating."""
import dataclasses

import numpy as np
import pytest

import golden_cases as G
from paper_2603_15202_b200.cluster import detector_classes
from paper_2603_15202_b200.config import DetectorConfig, PolicyConfig, UnsupportedConfigError
from paper_2603_15202_b200.hashing import chain_keys
from paper_2603_15202_b200.trace import class_key


@pytest.mark.parametrize("kb", [1, 2, 3])
def test_tracks_follow_first_arrival_and_class_key(kb):
    trace, _ = G.build("det_hot_n16")
    tid, off, ln, key = detector_classes(trace, kb)
    seen = {}
    for r in range(len(trace)):
        a, b = trace.blk_off[r], trace.blk_off[r + 1]
        k = class_key(trace.blocks[a:b].tolist(), kb)          # reference detector.py:41-45
        if k not in seen:
            seen[k] = len(seen)
            assert off[seen[k]] == a and ln[seen[k]] == min(kb, b - a)
        assert tid[r] == seen[k] and int(key[tid[r]]) == k
    # the exemplar is the class's leading chain keys (detector.py:305-306)
    r0 = int(np.nonzero(tid == 1)[0][0])
    blocks = trace.blocks[trace.blk_off[r0]:trace.blk_off[r0 + 1]].tolist()
    assert chain_keys(blocks)[:ln[1]] == chain_keys(blocks[:kb])


def test_empty_prefix_rejected():
    trace, _ = G.build("det_hot_n16")
    from paper_2603_15202_b200.trace import PackedTrace
    t = PackedTrace(trace.request_id[:2], trace.arrival_s[:2], trace.in_tokens[:2], trace.out_tokens[:2],
                    trace.class_key[:2], np.zeros(3, np.int64), np.zeros(0, np.uint64))
    with pytest.raises(ValueError):
        detector_classes(t, 2)


def test_detector_runs_with_every_policy():
    """Set-dependent scores included: filter (kept-set bs range) and uncapped linear (kept-set
    max batch size) have their own partials; only a non-device policy name is rejected."""
    _, cfg = G.build("det_hot_n16")
    for pol in (PolicyConfig(kind="linear"), PolicyConfig(kind="linear", bs_norm_cap=4), PolicyConfig(kind="filter"),
                PolicyConfig(kind="simulate"), PolicyConfig(kind="vllm"), PolicyConfig(kind="least_bs")):
        dataclasses.replace(cfg, policy=pol).check_device_supported()
    with pytest.raises(UnsupportedConfigError):
        dataclasses.replace(cfg, policy=dataclasses.replace(PolicyConfig(), kind="nope")).check_device_supported()


def test_detector_config_validation():
    with pytest.raises(ValueError):
        DetectorConfig(window_s=0).validate()
    with pytest.raises(ValueError):
        DetectorConfig(mitigation="nope").validate()
