"""§8f row 4 on the CPU: SampleBatch JSONL ingestion (rlo_batch_from_jsonl)
against the reference's own wire text (tests/golden/batch.jsonl, written by
SampleBatch::to_jsonl, sample.cpp:144-148) and its validation messages
(sample.cpp:85-102); bucket_plan (policy.cpp:542-548) against the reference."""
import json
import math
import os

import numpy as np
import pytest

import paper_2506_06122_b200 as rlo

G = os.path.join(os.path.dirname(__file__), "golden")


def _golden_text():
    with open(os.path.join(G, "batch.jsonl"), encoding="utf-8") as f:
        return f.read()


def _misc():
    with open(os.path.join(G, "misc.json")) as f:
        return json.load(f)


def _fnv1a(s):
    h = 0xcbf29ce484222325
    for c in s.encode("utf-8"):
        h = ((h ^ c) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_jsonl_matches_reference_records():
    text = _golden_text()
    recs = [json.loads(line) for line in text.splitlines() if line.strip()]  # independent parser
    b = rlo.batch_from_jsonl(text)
    B, T = b["B"], b["T"]
    assert B == len(recs) and T == max(1, max(len(r.get("response_tokens", [])) for r in recs))
    groups = {}
    first_missing = -1
    for i, r in enumerate(recs):
        n = len(r.get("response_tokens", []))
        assert b["lengths"][i] == n
        assert b["tokens"][i, :n].tolist() == r["response_tokens"]
        assert b["sample_keys"][i] == _fnv1a(r["sample_id"])
        assert b["group_index"][i] == groups.setdefault(r["group_id"], len(groups))
        m = r.get("action_mask", [])
        if b["mask"] is not None:
            assert b["mask"][i, :n].tolist() == (m if m else [1] * n)
        for k in ("response_logprobs", "ref_logprobs", "advantages"):
            if r.get(k):
                np.testing.assert_array_equal(b[k][i, :n], np.float32(r[k]))
        sr = r.get("scalar_reward")
        if sr is not None:
            assert b["scalar_rewards"][i] == np.float32(sr)
        elif b["scalar_rewards"] is not None:
            assert math.isnan(b["scalar_rewards"][i])
        if r.get("rewards"):
            np.testing.assert_array_equal(b["rewards"][i, :n], np.float32(r["rewards"]))
        elif sr is not None and n > 0 and b["rewards"] is not None:  # scalar on the last token, policy.cpp:268-270
            want = np.zeros(n, np.float32)
            want[-1] = np.float32(sr)
            np.testing.assert_array_equal(b["rewards"][i, :n], want)
        if n > 0 and not r.get("rewards") and sr is None and first_missing < 0:
            first_missing = i
    assert b["first_missing_reward"] == first_missing


@pytest.mark.parametrize("name", ["duplicate_id", "length_mismatch", "mask_mismatch"])
def test_jsonl_validation_messages_match_reference(name):
    code, msg, text = _misc()["jsonl_errors"][name]
    with pytest.raises(rlo.InputError) as e:
        rlo.batch_from_jsonl(text)
    assert code == 1 and str(e.value) == msg


def test_jsonl_malformed_is_input_error():
    with pytest.raises(rlo.InputError, match="malformed JSONL line 2"):
        rlo.batch_from_jsonl('{"sample_id":"a","response_tokens":[1]}\n{"sample_id": "b", "response_tokens": [1,}\n')
    b = rlo.batch_from_jsonl("\n\n")  # empty batch
    assert b["B"] == 0


def test_bucket_plan_matches_reference():
    for c in _misc()["bucket_plan"]:
        assert rlo.bucket_plan(c["total"], c["bucket"]) == c["plan"]
    assert rlo.bucket_plan(1000, 256) == [256, 256, 256, 232]  # test_policy.cpp:499-500
    with pytest.raises(rlo.ConfigError):
        rlo.bucket_plan(10, 0)


def test_jsonl_parallel_parse_reports_first_error_and_keeps_order(monkeypatch):
    """Large batches are parsed on several threads: the records keep their line
    order and the first malformed line (not the first one a thread meets) is
    the one reported, as the reference's sequential reader would."""
    lines = [json.dumps({"sample_id": f"s{i}", "group_id": f"g{i // 4}", "response_tokens": [i, i + 1, i + 2],
                         "scalar_reward": float(i % 3)}) for i in range(2000)]
    text = "\n".join(lines)
    for threads in ("1", "8"):
        monkeypatch.setenv("RLO_JSONL_THREADS", threads)
        b = rlo.batch_from_jsonl(text)
        assert b["B"] == 2000 and b["tokens"][1234].tolist() == [1234, 1235, 1236]
        assert b["group_index"][1999] == 499 and b["scalar_rewards"][5] == 2.0
    bad = list(lines)
    bad[1700] = '{"sample_id": "x", "response_tokens": [1,]}'
    bad[300] = '{"sample_id": "y", "response_tokens": [1, 2'
    monkeypatch.setenv("RLO_JSONL_THREADS", "8")
    with pytest.raises(rlo.InputError, match="malformed JSONL line 301:"):
        rlo.batch_from_jsonl("\n".join(bad))
