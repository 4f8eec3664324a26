"""Pins the CPU oracle (oracle/oracle.c) against the golden fixtures produced
by the reference's own code (tests/golden/make_golden.py -> oracle/_ref) and
against the reference's own known-answer tests
(/root/reference/proj/tests/test_policy.cpp, cited per test).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def test_logsoftmax_rows_match_reference():
    d = np.load(os.path.join(G, "logsoftmax.npz"))
    for off, V, tok, ref_lp in zip(d["offsets"], d["V"], d["tokens"], d["ref_lp"]):
        z = d["rows"][off:off + V].astype(np.float64)
        lse, _ = O.logsoftmax_row(z)
        assert abs((z[tok] - lse) - ref_lp) <= 1e-12 * max(1.0, abs(ref_lp))


def test_uniform_logits_give_minus_log_v():
    # test_policy.cpp:88-110: zero params -> every logp = -ln V (V=9), 1e-12
    lse, ent = O.logsoftmax_row(np.zeros(9))
    assert abs((0.0 - lse) + math.log(9.0)) < 1e-12
    assert abs(ent - math.log(9.0)) < 1e-12


def test_softmax_normalises():
    rng = np.random.default_rng(3)
    z = rng.standard_normal(1000) * 4
    lse, _ = O.logsoftmax_row(z)
    assert abs(np.exp(z - lse).sum() - 1.0) < 1e-9  # test_policy.cpp:101-109


def test_entropy_matches_definition():
    rng = np.random.default_rng(4)
    z = rng.standard_normal(777) * 3
    lse, ent = O.logsoftmax_row(z)
    p = np.exp(z - lse)
    assert abs(ent - float(-(p * (z - lse)).sum())) < 1e-10


def test_synthetic_generator_and_reference_lp():
    for c in load("logsoftmax_synth.json")["cases"]:
        row = O.synth_row(c["dtype"], c["V"], c["seed"], c["model"], c["key"])
        assert float(row.sum()) == c["row_sum"] and float(row.max()) == c["row_max"]
        assert O.synth_token(c["seed"], c["key"], c["V"]) == c["token"]
        lse, _ = O.logsoftmax_row(row)
        assert abs((row[c["token"]] - lse) - c["ref_lp"]) <= 1e-12 * max(1.0, abs(c["ref_lp"]))


def test_forward_logprobs_batch_and_oov():
    d = np.load(os.path.join(G, "forward_logprobs.npz"))
    row, lengths, tokens = d["row"], d["lengths"], d["tokens"]
    B, T, V = len(lengths), len(tokens) // len(lengths), row.size
    logits = np.tile(row, B * T)
    lp, _, tl = O.forward_logprobs(logits, O.F32, V, V, B, T, lengths, tokens)
    assert np.max(np.abs(lp - d["ref_lp"])) < 1e-12
    code, msg = load("misc.json")["oov_error"]
    with pytest.raises(O.OracleError) as e:
        O.forward_logprobs(logits, O.F32, V, V, B, T, lengths, d["bad_tokens"])
    assert e.value.code == code and str(e.value) == msg


def _arr(x, dt=np.float64):
    return None if x is None else np.asarray(x, dtype=dt)


def test_advantages_match_reference():
    for c in load("advantages.json")["cases"]:
        cfg = O.TrainConfig(**c["cfg"])
        args = (cfg, c["B"], c["T"], _arr(c["lengths"], np.int32), _arr(c["mask"], np.uint8),
                _arr(c["rewards_tok"]), _arr(c["rewards_seq"]))
        if c["error"]:
            with pytest.raises(O.OracleError) as e:
                O.compute_advantages(*args)
            assert [e.value.code, str(e.value)] == c["error"], c["name"]
        else:
            adv, _ = O.compute_advantages(*args)
            np.testing.assert_allclose(adv, c["ref_adv"], rtol=1e-12, atol=1e-12, err_msg=c["name"])


def test_advantages_bruteforce_discounted_sum():
    # test_policy.cpp:259-278: 1000 random sequences, T<=32, gamma 0.9, O(T^2) oracle, 1e-9
    rng = np.random.default_rng(314)
    cfg = O.TrainConfig(gamma=0.9, reward_clip=1e9, advantage_clip=1e9)
    for _ in range(1000):
        T = int(rng.integers(1, 33))
        r = rng.uniform(-1, 1, T)
        adv, _ = O.compute_advantages(cfg, 1, T, [T], rewards_tok=r)
        brute = [sum(0.9 ** (u - t) * r[u] for u in range(t, T)) for t in range(T)]
        assert np.max(np.abs(adv - brute)) < 1e-9


def test_whitening_normalises():
    # test_policy.cpp:281-304
    cfg = O.TrainConfig(whiten_advantages=1, advantage_clip=100.0)
    rt = np.concatenate([[0, 0, 0, float(i)] for i in range(4)])
    adv, _ = O.compute_advantages(cfg, 4, 4, [4] * 4, rewards_tok=rt)
    assert abs(adv.mean()) < 1e-9 and abs((adv ** 2).mean() - 1.0) < 1e-3


def _ppo_oracle(c, world=None):
    cfg = O.TrainConfig(**c["cfg"])
    V, B, T = c["V"], c["B"], c["T"]
    row = np.asarray(c["row"])
    lengths = np.asarray(c["lengths"], np.int32)
    tokens = np.asarray(c["tokens"], np.int32)
    lse, _ = O.logsoftmax_row(row)
    lp = row[tokens] - lse
    mask = _arr(c["mask"], np.uint8)
    world = world or c["world"]
    parts = []
    sizes = O.split_sizes(B, world)
    off = 0
    for s in sizes:  # ppo_update's split_batch sharding, policy.cpp:465-469
        sl = slice(off * T, (off + s) * T)
        _, _, p = O.ppo_loss(cfg, int(s), T, lengths[off:off + s], None if mask is None else mask[sl], lp[sl],
                             np.asarray(c["old"])[sl], None if c["ref"] is None else np.asarray(c["ref"])[sl],
                             np.asarray(c["adv"])[sl])
        parts.append(p)
        off += s
    return O.merge(np.array(parts), cfg)


def test_ppo_stats_match_reference():
    d = load("ppo_stats.json")
    for c in d["cases"]:
        st = _ppo_oracle(c)
        for k in ["loss", "mean_ratio", "clip_fraction", "mean_kl"]:
            assert abs(st[k] - c["ref_stats"][k]) <= 1e-12 * max(1.0, abs(c["ref_stats"][k])), k
        assert st["tokens"] == c["ref_stats"]["tokens"]
    kat = d["cases"][-1]
    assert abs(_ppo_oracle(kat)["loss"] - (-(1.0 + 0.2) * 2.0)) < 1e-12  # test_policy.cpp:373-374


def test_ppo_error_paths_match_reference():
    errs = load("ppo_stats.json")["errors"]
    cfg = O.TrainConfig()
    _, _, p = O.ppo_loss(cfg, 1, 1, [1], [0], [-1.0], [-1.0], None, [0.5])
    with pytest.raises(O.OracleError) as e:
        O.merge(p[None], cfg)
    assert [e.value.code, str(e.value)] == errs["no_tokens"]
    _, _, p = O.ppo_loss(cfg, 1, 1, [1], None, [-1.0], [-1.0], None, [float("nan")])
    with pytest.raises(O.OracleError) as e:
        O.merge(p[None], cfg)
    assert [e.value.code, str(e.value)] == errs["nan_adv"]


def test_ratio_one_identity():
    # test_policy.cpp:339-355: old == lp, kl_coef 0 -> loss == -mean(A)
    rng = np.random.default_rng(21)
    B, T = 5, 6
    lp = rng.uniform(-5, -0.1, B * T)
    adv = rng.uniform(-1, 1, B * T)
    cfg = O.TrainConfig()
    _, _, p = O.ppo_loss(cfg, B, T, [T] * B, None, lp, lp, None, adv)
    assert abs(O.merge(p[None], cfg)["loss"] + adv.mean()) < 1e-12


def test_clip_monotonicity():
    # test_policy.cpp:439-452
    rng = np.random.default_rng(71)
    B, T = 4, 5
    lp = rng.uniform(-3, -0.1, B * T)
    adv = rng.uniform(-1, 1, B * T)
    prev = math.inf
    for eps in [0.05, 0.1, 0.2, 0.4, 0.8]:
        cfg = O.TrainConfig(clip_eps=eps)
        _, _, p = O.ppo_loss(cfg, B, T, [T] * B, None, lp, lp, None, adv)
        loss = O.merge(p[None], cfg)["loss"]
        assert loss <= prev + 1e-12
        prev = loss


def test_split_sizes_match_reference():
    for c in load("misc.json")["split_sizes"]:
        assert O.split_sizes(c["n"], c["parts"]).tolist() == c["sizes"]


def test_dual_clip_and_kl_estimators_definitions():
    # extensions (parity unpinned by the reference): direct restatement checks
    cfg = O.TrainConfig(dual_clip_c=3.0, kl_coef=0.1, kl_estimator=O.K3)
    lp = np.array([-1.0, -1.0])
    old = np.array([-3.0, -1.1])  # ratio e^2 (A<0 -> dual clip), ~1.105
    ref = np.array([-1.2, -0.7])
    adv = np.array([-1.0, 0.5])
    loss_tok, dlogp, p = O.ppo_loss(cfg, 1, 2, [2], None, lp, old, ref, adv)
    r = lp - ref
    k3 = np.exp(-r) - 1 + r
    assert abs(loss_tok[0] - (3.0 * 1.0 + 0.1 * k3[0])) < 1e-12  # capped at -c*A
    assert abs(dlogp[0] - 0.1 * (1 - np.exp(-r[0]))) < 1e-12       # dual branch: no pg gradient
    ratio1 = math.exp(0.1)
    assert abs(loss_tok[1] - (-min(ratio1 * 0.5, min(ratio1, 1.2) * 0.5) + 0.1 * k3[1])) < 1e-12
    assert p[O.NPARTIAL - 11] == 1.0  # RLO_P_DUAL_CLIPPED == 5


def test_grpo_and_gae_definitions():
    cfg = O.TrainConfig(adv_estimator=O.GRPO, group_size=4, advantage_clip=100.0)
    R = np.array([1.0, 0.0, 1.0, 1.0, 0.0, 0.0, 0.0, 0.0])
    adv, _ = O.compute_advantages(cfg, 8, 3, [3, 2, 3, 1, 3, 3, 3, 0], rewards_seq=R)
    g = R[:4]
    a0 = (g - g.mean()) / (g.std() + 1e-6)
    assert abs(adv[0] - a0[0]) < 1e-12 and abs(adv[3] - a0[1]) < 1e-12 and adv[5] == 0.0
    assert np.all(adv[12:] == 0.0)  # all-equal group -> 0
    cfg = O.TrainConfig(adv_estimator=O.GAE, gamma=0.99, lambd=0.95, advantage_clip=100.0)
    rng = np.random.default_rng(5)
    T = 7
    r = rng.standard_normal(T)
    v = rng.standard_normal(T)
    adv, ret = O.compute_advantages(cfg, 1, T, [T], rewards_tok=r, values=v)
    vn = np.append(v[1:], 0.0)
    delta = r + 0.99 * vn - v
    brute = [sum((0.99 * 0.95) ** (u - t) * delta[u] for u in range(t, T)) for t in range(T)]
    assert np.max(np.abs(adv - brute)) < 1e-12 and np.max(np.abs(ret - (adv + v))) < 1e-12


def _ext():
    with open(os.path.join(G, "extensions.json")) as f:
        return json.load(f)


def test_gae_lambda1_is_reference_return_minus_value():
    """GAE (an extension) pinned to the reference: lambda = 1 telescopes to the
    reference's discounted return minus the critic value."""
    for c in _ext()["gae_lambda1"]:
        adv, _ = O.compute_advantages(O.TrainConfig(**c["cfg"]), c["B"], c["T"], c["lengths"], c["mask"],
                                      rewards_tok=c["rewards_tok"], values=c["values"])
        np.testing.assert_allclose(adv, c["expect"], rtol=1e-9, atol=1e-9)


def test_grpo_one_group_is_reference_whitening():
    """GRPO (an extension) pinned to the reference: one group of one-token
    samples with eps = 1e-8 is the reference's whitening of the rewards."""
    for c in _ext()["grpo_one_group"]:
        adv, _ = O.compute_advantages(O.TrainConfig(**c["cfg"]), c["B"], c["T"], c["lengths"],
                                      rewards_seq=c["rewards_seq"])
        np.testing.assert_allclose(adv, c["expect"], rtol=1e-9, atol=1e-12)


def test_entropy_is_reference_softmax_entropy():
    """Entropy (an extension) pinned to the reference's own full log-softmax."""
    for c in _ext()["entropy"]:
        _, h = O.logsoftmax_row(np.asarray(c["row"], np.float64))
        assert abs(h - c["entropy"]) <= 1e-11 * max(1.0, abs(c["entropy"])), c["V"]


def test_aggregation_and_dual_clip_identities_match_reference():
    """seq-mean-token-mean and group-mean on equal-length unmasked batches, and
    a never-binding dual-clip cap, reproduce the reference's token-mean loss."""
    for c in _ext()["aggregation"]:
        B, T = c["B"], c["T"]
        lp = np.asarray(O.ref_logsoftmax_rows(np.asarray(c["row"]), [0], full=True)[1][0])[np.asarray(c["tokens"])]
        for extra in (dict(loss_agg=1), dict(loss_agg=3, group_size=c["G"]), dict(dual_clip_c=1e9)):
            oc = O.TrainConfig(**c["cfg"], **extra)
            _, _, part = O.ppo_loss(oc, B, T, c["lengths"], None, lp, c["old"], c["ref"], c["adv"], np.zeros(B * T))
            got = O.merge(part[None], oc)
            assert abs(got["loss"] - c["ref_stats"]["loss"]) <= 1e-12 * max(1.0, abs(c["ref_stats"]["loss"])), extra
