"""Oracle pinning for the §8f "next" rows (CPU): the actor backward epilogue
and the critic value loss against the reference's own gradients
(tests/golden: ppo_gradient -> merge_gradients b2-segment, value_gradient)."""
import json
import os

import numpy as np

import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def _load(n):
    with open(os.path.join(G, n)) as f:
        return json.load(f)


def test_backward_rows_sum_to_reference_gradient():
    for c in _load("ppo_stats.json")["cases"]:
        if "ref_grad_row" not in c:
            continue
        cfg = O.TrainConfig(**c["cfg"])
        B, T = c["B"], c["T"]
        row = np.asarray(c["row"])
        toks = np.asarray(c["tokens"], np.int32)
        lengths = np.asarray(c["lengths"], np.int32)
        mask = None if c["mask"] is None else np.asarray(c["mask"], np.uint8)
        lse, _ = O.logsoftmax_row(row)
        lp = row[toks] - lse
        ref = None if c["ref"] is None else np.asarray(c["ref"])
        _, dl, _ = O.ppo_loss(cfg, B, T, lengths, mask, lp, np.asarray(c["old"]), ref, np.asarray(c["adv"]))
        w = O.loss_weights(cfg, B, T, lengths, mask)
        g = np.zeros(row.size)
        for i in range(B * T):
            if w[i] * dl[i] != 0.0:
                g += O.logits_backward_row(row, int(toks[i]), w[i] * dl[i])
        np.testing.assert_allclose(g, c["ref_grad_row"], rtol=1e-10, atol=1e-13)


def test_value_loss_matches_reference():
    for c in _load("value_loss.json")["cases"]:
        B, T = c["B"], c["T"]
        mask = None if c["mask"] is None else np.asarray(c["mask"], np.uint8)
        dv, o = O.value_loss(B, T, np.asarray(c["lengths"], np.int32), mask, np.full(B * T, c["vb"]), None,
                             np.asarray(c["targets"]))
        assert abs(o["loss_sum"] - c["ref"]["loss_sum"]) <= 1e-12 * max(1.0, abs(c["ref"]["loss_sum"]))
        assert o["tokens"] == c["ref"]["tokens"]
        assert abs(dv.sum() - c["ref"]["grad_vb"]) <= 1e-12 * max(1.0, abs(c["ref"]["grad_vb"]))


def test_loss_weights_sum_to_one_per_unit():
    rng = np.random.default_rng(2)
    B, T = 12, 9
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[0] = T
    mask = (rng.random(B * T) < 0.7).astype(np.uint8)
    for agg in range(4):
        w = O.loss_weights(O.TrainConfig(loss_agg=agg, group_size=3), B, T, lengths, mask)
        if agg == 2:  # seq-mean-token-sum: each non-empty sequence sums to its token count / seqs
            continue
        assert abs(w.sum() - 1.0) < 1e-12, agg


def test_decode_next_matches_reference():
    d = _load("decode.json")
    for c in d["cases"]:
        tok, lp = O.decode_next(np.asarray(d["rows"][c["row"]]), c["temperature"], c["seed"], c["version"],
                                c["sample_key"], c["position"])
        assert tok == c["ref_token"] and abs(lp - c["ref_logp"]) <= 1e-12
        assert O.hash_str(c["sample_id"]) == c["sample_key"]


def test_sample_key_is_reference_hash():
    import paper_2506_06122_b200 as rlo
    d = _load("decode.json")
    for c in d["cases"][:20]:
        assert rlo.sample_key(c["sample_id"]) == c["sample_key"]
