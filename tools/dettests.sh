#!/bin/bash
# run detector-related GPU tests one by one with a hard timeout
cd "$1"
for t in "test_replay_matches_reference_golden[det_api_k1]" "test_replay_matches_reference_golden[det_chat_default]" "test_replay_matches_reference_golden[det_evict_n8]" "test_replay_matches_reference_golden[det_hot_force_mean]" "test_replay_matches_reference_golden[det_hot_n16]" "test_replay_matches_reference_golden[det_hot_vllm_stale]" "test_random_detector_configs_match_oracle"; do
  s=$(date +%s)
  timeout 90 python -m pytest -q -x "tests/test_device_parity.py::$t" -m gpu > /tmp/o.log 2>&1
  rc=$?
  e=$(date +%s)
  echo "$t rc=$rc dt=$((e - s))"
  [ $rc -ne 0 ] && tail -5 /tmp/o.log
done
