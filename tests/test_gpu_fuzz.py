"""Randomised GPU parity sweep: many small whole-path cases drawn from one
seeded generator — vocabulary sizes (odd ones too), padded / unaligned row
strides, fp32 / bf16, P = 1..3 logits tensors, ragged lengths including empty
responses, masks, every estimator / KL estimator / aggregation, dual-clip and
whitening — each checked against the fp64 oracle (advantages, per-token
log-probs / entropy / loss, merged stats)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2506_06122_b200 as rlo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, rlo, rlo.Objective(0)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def close_arr(got, want, tol, what):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    assert np.all(err <= tol), f"{what}: max scaled err {err.max():.3g}"


@pytest.mark.parametrize("case", range(64))
def test_random_whole_path_vs_oracle(env, case):
    torch, rlo, obj = env
    rng = np.random.default_rng(9000 + case)
    est = ["reinforce", "grpo", "gae"][case % 3]
    G = int(rng.choice([1, 2, 4])) if est == "grpo" else 1
    B = G * int(rng.integers(1, 5)) if est == "grpo" else int(rng.integers(1, 9))
    T = int(rng.integers(1, 17))
    V = int(rng.choice([1, 7, 64, 1000, 2049, 4099, 8192]))
    dtype = O.BF16 if case % 4 == 3 else O.F32
    P = int(rng.integers(1, 4))
    pad = int(rng.choice([0, 1, 8]))
    stride = V + pad
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[0] = max(1, lengths[0])
    masked = bool(rng.random() < 0.5)
    mask = (rng.random((B, T)) < 0.8).astype(np.uint8) if masked else None
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    cfg_kw = dict(adv_estimator=est, group_size=G, gamma=float(rng.choice([1.0, 0.95])), lambd=0.9,
                  whiten_advantages=bool(rng.random() < 0.5), kl_coef=float(rng.choice([0.0, 0.02])),
                  kl_estimator=str(rng.choice(["k1", "k2", "k3"])), dual_clip_c=float(rng.choice([0.0, 3.0])),
                  loss_agg=int(rng.integers(0, 4)), clip_eps=float(rng.choice([0.1, 0.2])),
                  reward_clip=float(rng.choice([20.0, 1.0])), advantage_clip=float(rng.choice([10.0, 2.0])))
    cfg = rlo.TrainConfig(**cfg_kw)
    oc = O.TrainConfig(**{**cfg_kw, "adv_estimator": {"reinforce": 0, "grpo": 1, "gae": 2}[est],
                          "kl_estimator": {"k1": 0, "k2": 1, "k3": 2}[cfg_kw["kl_estimator"]],
                          "whiten_advantages": int(cfg_kw["whiten_advantages"])})
    # rewards / values
    rw_tok = rw_seq = vals = None
    if est == "grpo" or rng.random() < 0.5:
        rw_seq = (rng.random(B) < 0.5).astype(np.float32) + rng.standard_normal(B).astype(np.float32) * 0.1
    else:
        rw_tok = (rng.standard_normal((B, T)) * 0.5).astype(np.float32)
    if est == "gae":
        vals = (rng.standard_normal((B, T)) * 0.5).astype(np.float32)
    # logits rows (padded stride, garbage in the padding)
    base = (rng.standard_normal((B * T, stride)) * 2.5).astype(np.float32)
    rows = [base]
    for _ in range(P - 1):
        rows.append((base + rng.standard_normal((B * T, stride)).astype(np.float32) * 0.2).astype(np.float32))
    for r in rows:
        r[:, V:] = np.nan
    tdt = torch.float32 if dtype == O.F32 else torch.bfloat16
    dev_rows = [dev(torch, r).to(tdt)[:, :V] for r in rows]
    if dtype == O.BF16:  # the oracle reads the bf16-rounded values
        host_rows = [np.ascontiguousarray(t.float().cpu().numpy()) for t in dev_rows]
        host_stride = V
    else:
        host_rows, host_stride = rows, stride
    # advantages
    L, M = dev(torch, lengths), (dev(torch, mask) if mask is not None else None)
    adv = obj.compute_advantages(cfg, L, T=T, mask=M, rewards=None if rw_tok is None else dev(torch, rw_tok),
                                 scalar_rewards=None if rw_seq is None else dev(torch, rw_seq),
                                 values=None if vals is None else dev(torch, vals))
    oadv, _ = O.compute_advantages(oc, B, T, lengths, None if mask is None else mask.ravel(),
                                   rewards_tok=None if rw_tok is None else rw_tok.ravel(),
                                   rewards_seq=rw_seq, values=None if vals is None else vals.ravel())
    valid = (np.arange(T)[None, :] < lengths[:, None]).ravel()
    close_arr(adv.cpu().numpy().ravel()[valid], oadv[valid], 2e-5, f"advantages case {case}")
    # loss pass
    old_lp = ref_lp = None
    kw = {}
    if P >= 2:
        kw["old_logits"] = dev_rows[1]
    else:
        old_lp = rng.uniform(-9, -1, (B, T)).astype(np.float32)
        kw["old_logprobs"] = dev(torch, old_lp)
    if P >= 3:
        kw["ref_logits"] = dev_rows[2]
    else:
        ref_lp = rng.uniform(-9, -1, (B, T)).astype(np.float32)
        kw["ref_logprobs"] = dev(torch, ref_lp)
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), L, dev_rows[0], adv, mask=M,
                            outputs=("logp", "entropy", "loss", "dlogp"), **kw)
    valid = (np.arange(T)[None, :] < lengths[:, None]).ravel()
    m = valid & (np.ones(B * T, bool) if mask is None else mask.ravel() != 0)
    if not m.any():  # policy.cpp:437
        with pytest.raises(rlo.TrainingError, match="no loss-participating tokens"):
            obj.merge_gradients(cfg)
        return
    st = obj.merge_gradients(cfg)
    lps = [O.forward_logprobs(host_rows[k], O.F32, V, host_stride, B, T, lengths, tokens) for k in range(P)]
    o_old = lps[1][0] if P >= 2 else old_lp.ravel().astype(np.float64)
    o_ref = lps[2][0] if P >= 3 else ref_lp.ravel().astype(np.float64)
    loss_tok, dlogp, part = O.ppo_loss(oc, B, T, lengths, None if mask is None else mask.ravel(), lps[0][0], o_old,
                                       o_ref, adv.cpu().numpy().ravel(), lps[0][1])
    close_arr(outs["logp"].cpu().numpy().ravel()[m], lps[0][0][m], TOL, f"logp case {case}")
    close_arr(outs["entropy"].cpu().numpy().ravel()[m], lps[0][1][m], 2e-5, f"entropy case {case}")
    close_arr(outs["loss"].cpu().numpy().ravel()[m], loss_tok[m], 2e-5, f"loss case {case}")
    close_arr(outs["dlogp"].cpu().numpy().ravel()[m], dlogp[m], 2e-5, f"dlogp case {case}")
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert abs(getattr(st, k) - want[k]) <= 2e-5 * max(1.0, abs(want[k])), (case, k, getattr(st, k), want[k])
    for k in ("tokens", "seqs", "groups"):
        assert getattr(st, k) == want[k], (case, k)


@pytest.mark.parametrize("case", range(16))
def test_random_update_pass_vs_oracle(env, case):
    """Fused / two-pass actor update (whichever the entry picks) on random
    shapes, padded or packed logits: gradient rows vs the oracle's
    w*dlogp*(onehot - softmax), untouched padding."""
    torch, rlo, obj = env
    rng = np.random.default_rng(7000 + case)
    B, T = int(rng.integers(1, 7)), int(rng.integers(1, 9))
    V = int(rng.choice([8, 1000, 4096, 32000]))
    dtype = torch.float32 if case % 3 else torch.bfloat16
    P = int(rng.integers(1, 4))
    packed = bool(case % 2)
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[0] = max(1, lengths[0])
    mask = (rng.random((B, T)) < 0.85).astype(np.uint8)
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    adv = rng.uniform(-1.5, 1.5, (B, T)).astype(np.float32)
    gen = torch.Generator().manual_seed(case)
    full = [(torch.randn(B * T, V, generator=gen) * 2).to(dtype)]
    for _ in range(P - 1):
        full.append((full[0].float() + torch.randn(B * T, V, generator=gen) * 0.1).to(dtype))
    valid = np.concatenate([np.arange(b * T, b * T + lengths[b]) for b in range(B)])
    start = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    x = [(t[torch.from_numpy(valid)] if packed else t).contiguous().cuda() for t in full]
    cfg = rlo.TrainConfig(loss_agg=int(rng.integers(0, 4)), group_size=1, kl_coef=0.01, kl_estimator="k3")
    L, K, M, A = dev(torch, lengths), dev(torch, tokens), dev(torch, mask), dev(torch, adv)
    cnt = obj.batch_counts(cfg, L, T, mask=M)
    if cnt.tokens == 0:
        return
    w = obj.loss_weights(cfg, L, cnt, T, mask=M)
    kw = dict(old_logits=x[1]) if P >= 2 else dict(old_logprobs=dev(torch, np.full((B, T), -6.0, np.float32)))
    if P >= 3:
        kw["ref_logits"] = x[2]
    else:
        kw["ref_logprobs"] = dev(torch, np.full((B, T), -6.0, np.float32))
    nrows = len(valid) if packed else B * T
    g = torch.full((nrows + 2, V), 777.0, device="cuda")
    outs, _ = obj.ppo_gradient_fused(cfg, K, L, x[0], A, w, mask=M, grad=g[:nrows], outputs=("dlogp",),
                                     seq_start=dev(torch, start) if packed else None, **kw)
    obj.merge_gradients(cfg)
    assert bool((g[nrows:] == 777.0).all())
    G = g[:nrows].cpu().numpy()
    rows = full[0].float().numpy().astype(np.float64)
    dl, wv = outs["dlogp"].cpu().numpy().ravel(), w.cpu().numpy().ravel()
    for j, r in enumerate(valid if packed else range(B * T)):
        scale = float(np.float32(wv[r]) * np.float32(dl[r]))
        if scale == 0.0:
            assert not G[j].any()
            continue
        want = O.logits_backward_row(rows[r], int(tokens.ravel()[r]), scale)
        assert np.abs(G[j] - want).max() <= 1e-5 * abs(scale) + 1e-12, (case, j)


@pytest.mark.parametrize("case", range(24))
def test_random_long_rows_loss_pass_vs_oracle(env, case):
    """Long bf16 rows (the lockstep kernels on a deferred offset for P = 2 / 3,
    two rows per warp for P = 1): random vocabularies >= 64 Ki (odd ones,
    padded and unaligned strides), old / ref rows shifted against the actor
    by up to +-90 nats, -inf masked entries, late spikes far above a thread's
    first batch, whole rows shifted by hundreds of nats -- per-token log-probs
    of every tensor and the entropy against the fp64 oracle."""
    torch, rlo, obj = env
    rng = np.random.default_rng(12000 + case)
    V = int(rng.choice([65536, 65537, 100003, 131072, 152064]))
    pad = int(rng.choice([0, 8, 1]))
    stride = V + pad
    P = [1, 2, 3][case % 3]
    B, T = int(rng.integers(1, 4)), int(rng.integers(1, 5))
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    n = B * T
    base = (rng.standard_normal((n, stride)) * float(rng.choice([1.0, 2.5, 4.0]))).astype(np.float32)
    if rng.random() < 0.3:
        base += float(rng.choice([-300.0, 150.0, 400.0]))
    if rng.random() < 0.4:  # late spikes, far above the thread's first batch
        for r in range(n):
            base[r, int(rng.integers(V // 2, V))] += float(rng.choice([20.0, 45.0, 90.0]))
    masked = rng.random() < 0.3
    if masked:  # masked vocabulary entries, the same in every tensor
        idx = rng.choice(V, V // 5, replace=False)
        base[:, idx] = -np.inf
    rows = [base]
    for _ in range(P - 1):
        off = float(rng.choice([0.0, 5.0, -5.0, 30.0, -30.0, 90.0, -90.0]))
        rows.append((base + off + rng.standard_normal((n, stride)).astype(np.float32) * 0.3).astype(np.float32))
    dev_rows = [dev(torch, r).to(torch.bfloat16)[:, :V] for r in rows]
    host_rows = [np.ascontiguousarray(t.float().cpu().numpy()) for t in dev_rows]
    tokens = np.zeros((B, T), np.int32)
    for r in range(n):  # a finite logit (masked entries hold -inf)
        fin = np.flatnonzero(np.isfinite(host_rows[0][r]))
        tokens.ravel()[r] = int(rng.choice(fin))
    cfg = rlo.TrainConfig(kl_coef=0.001, kl_estimator="k3")
    kw = {}
    kw.update(old_logits=dev_rows[1]) if P >= 2 else kw.update(
        old_logprobs=dev(torch, rng.uniform(-9, -1, (B, T)).astype(np.float32)))
    kw.update(ref_logits=dev_rows[2]) if P >= 3 else kw.update(
        ref_logprobs=dev(torch, rng.uniform(-9, -1, (B, T)).astype(np.float32)))
    adv = dev(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32))
    names = ("logp", "old_logp", "ref_logp")[:P]
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), dev_rows[0], adv,
                            outputs=names + ("entropy",), **kw)
    try:
        obj.merge_gradients(cfg)
    except rlo.TrainingError:  # ratios of rows shifted far apart can overflow, as in the reference
        pass
    m = (np.arange(T)[None, :] < lengths[:, None]).ravel()
    for k, name in enumerate(names):
        lp, ent, _ = O.forward_logprobs(host_rows[k], O.F32, V, V, B, T, lengths, tokens)
        close_arr(outs[name].cpu().numpy().ravel()[m], lp[m], TOL, f"{name} case {case} V {V} pad {pad} P {P}")
        if k == 0:
            close_arr(outs["entropy"].cpu().numpy().ravel()[m], ent[m], 2e-5, f"entropy case {case}")
