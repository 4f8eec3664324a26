"""GPU parity of the fused update pass (rlo_ppo_gradient_fused): the loss
pass and the actor backward epilogue in one read of the actor logits
(policy.cpp:355-379).  Checked against the oracle row by row and against the
two-pass form (rlo_ppo_gradient + rlo_logits_backward) it replaces, plus
rlo_batch_counts against the counts merge_gradients derives."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2506_06122_b200 as rlo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, rlo, rlo.Objective(0)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _case(torch, seed, B, T, V, dt, P, G=3):
    rng = np.random.default_rng(seed)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    gen = torch.Generator().manual_seed(seed)
    x = [(torch.randn(B * T, V, generator=gen) * 3).to(tdt).cuda()]
    for _ in range(P - 1):  # old / ref: the actor plus a small perturbation
        x.append((x[0].float() + torch.randn(B * T, V, generator=gen).cuda() * 0.05).to(tdt))
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    mask = (rng.random((B, T)) < 0.85).astype(np.uint8)
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    adv = rng.uniform(-1.5, 1.5, (B, T)).astype(np.float32)
    old = rng.uniform(-12, -4, (B, T)).astype(np.float32)
    ref = rng.uniform(-12, -4, (B, T)).astype(np.float32)
    return x, lengths, mask, toks, adv, old, ref


def _kw(torch, P, x, old, ref):
    kw = {}
    if P >= 2:
        kw["old_logits"] = x[1]
    else:
        kw["old_logprobs"] = dev(torch, old)
    if P >= 3:
        kw["ref_logits"] = x[2]
    else:
        kw["ref_logprobs"] = dev(torch, ref)
    return kw


@pytest.mark.parametrize("dt,gdt,V,P", [
    ("f32", "f32", 32000, 3),   # cfg 1-2 vocabulary: 2-CTA cluster
    ("f32", "f32", 4099, 1),    # odd V: the last slice's scalar tail
    ("f32", "f32", 10000, 2),   # 2-CTA cluster
    ("f32", "bf16", 20008, 3),  # 4-CTA cluster, uneven last slice
    ("f32", "bf16", 5000, 2),
    ("bf16", "bf16", 152064, 3),  # Qwen2.5 vocabulary: 4-CTA cluster
    ("bf16", "f32", 2051, 1),
])
@pytest.mark.parametrize("agg", [0, 1, 3])
def test_fused_matches_two_pass_and_oracle(env, dt, gdt, V, P, agg):
    torch, rlo, obj = env
    B, T = 6, 5
    x, lengths, mask, toks, adv, old, ref = _case(torch, agg * 7 + P, B, T, V, dt, P)
    gtdt = torch.float32 if gdt == "f32" else torch.bfloat16
    cfg = rlo.TrainConfig(loss_agg=agg, group_size=3, kl_coef=0.01, kl_estimator="k3")
    L, K, M, A = dev(torch, lengths), dev(torch, toks), dev(torch, mask), dev(torch, adv)
    kw = _kw(torch, P, x, old, ref)
    # two-pass reference form
    outs2 = obj.ppo_gradient(cfg, K, L, x[0], A, mask=M, outputs=("logp", "dlogp", "lse", "entropy", "loss"), **kw)
    st2 = obj.merge_gradients(cfg)
    w = obj.loss_weights(cfg, L, st2, T, mask=M)
    g2 = obj.logits_backward(K, L, x[0], outs2["lse"], outs2["dlogp"], w, grad_dtype=gtdt)
    # counts ahead of the pass == the merged counts
    cnt = obj.batch_counts(cfg, L, T, mask=M)
    assert (cnt.tokens, cnt.seqs, cnt.groups) == (st2.tokens, st2.seqs, st2.groups)
    w1 = obj.loss_weights(cfg, L, cnt, T, mask=M)
    assert torch.equal(w, w1)
    # fused
    n0 = rlo.launch_count()
    outs1, g1 = obj.ppo_gradient_fused(cfg, K, L, x[0], A, w1, mask=M, grad_dtype=gtdt,
                                       outputs=("logp", "dlogp", "lse", "entropy", "loss"), **kw)
    if (dt, V) == ("f32", 32000):
        assert rlo.launch_count() - n0 == 2  # the one-pass kernel (+ per-sequence reduce), not the two-pass form
    st1 = obj.merge_gradients(cfg)
    for k in ("logp", "dlogp", "entropy", "loss"):
        a, b = outs1[k].cpu().numpy(), outs2[k].cpu().numpy()
        assert np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))) <= 2e-6, k
    assert st1.tokens == st2.tokens and st1.clip_fraction == st2.clip_fraction
    for f in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert abs(getattr(st1, f) - getattr(st2, f)) <= 2e-6 * max(1.0, abs(getattr(st2, f))), f
    # gradient rows: fused vs the oracle (fp64) and vs the two-pass kernel
    G1, G2 = g1.float().cpu().numpy(), g2.float().cpu().numpy()
    rows = x[0].float().cpu().numpy()
    dl, wv = outs1["dlogp"].cpu().numpy().ravel(), w1.cpu().numpy().ravel()
    tol = 1e-5 if gdt == "f32" else 8e-3
    for i in range(B * T):
        scale = float(np.float32(wv[i]) * np.float32(dl[i]))
        if scale == 0.0:
            assert not G1[i].any(), i
            continue
        want = O.logits_backward_row(rows[i].astype(np.float64), int(toks.ravel()[i]), scale)
        assert np.abs(G1[i] - want).max() <= tol * abs(scale) + 1e-12, (i, np.abs(G1[i] - want).max(), scale)
        assert np.abs(G1[i] - G2[i]).max() <= 2 * tol * abs(scale) + 1e-12, i


def test_fused_kernel_forced_for_bf16_qwen_vocab(env, monkeypatch):
    """The bf16 Qwen row runs two-pass by default (measured faster); force the
    8-CTA cluster kernel and check it against the same oracle."""
    torch, rlo, _ = env
    monkeypatch.setenv("RLO_FUSED_SLICE_KB", "40")  # knobs are read when a handle is created
    test_fused_matches_two_pass_and_oracle((torch, rlo, rlo.Objective(0)), "bf16", "bf16", 152064, 3, 1)
    monkeypatch.setenv("RLO_FUSED_SLICE_KB", "16")  # 8 CTAs x 19 KB, fp32 with a bf16 gradient
    test_fused_matches_two_pass_and_oracle((torch, rlo, rlo.Objective(0)), "f32", "bf16", 32000, 2, 3)


def test_fused_micro_batches_and_neg_inf(env):
    """Micro-batches accumulate like ppo_gradient; -inf logits take the guarded
    entropy redo from shared memory."""
    torch, rlo, obj = env
    B, T, V = 6, 4, 32000
    x, lengths, mask, toks, adv, old, ref = _case(torch, 11, B, T, V, "f32", 1)
    x0 = x[0].clone()
    x0[3, 100:20000] = float("-inf")
    x0[7, :] = float("-inf")
    x0[7, toks.ravel()[7]] = 1.0  # only the token survives
    cfg = rlo.TrainConfig()
    L, K, M, A, OL = (dev(torch, v) for v in (lengths, toks, mask, adv, old))
    cnt = obj.batch_counts(cfg, L, T, mask=M)
    w = obj.loss_weights(cfg, L, cnt, T, mask=M)
    outs, g = obj.ppo_gradient_fused(cfg, K, L, x0, A, w, mask=M, old_logprobs=OL, outputs=("logp", "entropy"))
    st1 = obj.merge_gradients(cfg)
    grads = []
    for s0 in (3, 0):
        rs = slice(s0 * T, (s0 + 3) * T)
        _, gm = obj.ppo_gradient_fused(cfg, K[s0:s0 + 3], L[s0:s0 + 3], x0[rs], A[s0:s0 + 3], w[s0:s0 + 3],
                                       mask=M[s0:s0 + 3], old_logprobs=OL[s0:s0 + 3], seq_offset=s0)
        grads.append((rs, gm))
    st2 = obj.merge_gradients(cfg)
    assert st1 == st2
    for rs, gm in grads:
        assert torch.equal(gm, g[rs])
    ent = outs["entropy"].cpu().numpy().ravel()
    assert np.all(np.isfinite(ent))
    rows = x0.double().cpu().numpy()
    for i in (3, 7):
        if w.cpu().numpy().ravel()[i] == 0:
            continue
        lse, h = O.logsoftmax_row(rows[i])
        assert abs(outs["logp"].cpu().numpy().ravel()[i] - (rows[i, toks.ravel()[i]] - lse)) <= 1e-5
        assert abs(ent[i] - h) <= 2e-5 * max(1.0, h)
    assert torch.isfinite(g).all()


def test_fused_unaligned_rows_take_two_pass(env):
    """A row stride that breaks 16-byte alignment falls back to the two-pass
    form with identical results."""
    torch, rlo, obj = env
    B, T, V = 3, 4, 1001
    x, lengths, mask, toks, adv, old, ref = _case(torch, 5, B, T, V + 1, "f32", 1)
    xs = x[0][:, 1:]  # stride V+1, base offset 4 bytes: not 16-byte aligned
    toks = np.minimum(toks, V - 1)
    cfg = rlo.TrainConfig()
    L, K, M, A, OL = (dev(torch, v) for v in (lengths, toks, mask, adv, old))
    cnt = obj.batch_counts(cfg, L, T, mask=M)
    w = obj.loss_weights(cfg, L, cnt, T, mask=M)
    outs, g = obj.ppo_gradient_fused(cfg, K, L, xs, A, w, mask=M, old_logprobs=OL, grad_dtype=torch.float32)
    obj.merge_gradients(cfg)
    outs2 = obj.ppo_gradient(cfg, K, L, xs.contiguous(), A, mask=M, old_logprobs=OL, outputs=("dlogp", "lse"))
    obj.merge_gradients(cfg)
    g2 = obj.logits_backward(K, L, xs.contiguous(), outs2["lse"], outs2["dlogp"], w, grad_dtype=torch.float32)
    assert torch.allclose(g, g2, rtol=1e-5, atol=1e-9)


def test_fused_errors(env):
    torch, rlo, obj = env
    B, T, V = 2, 3, 64
    x = torch.zeros(B * T, V, device="cuda")
    L = dev(torch, np.array([3, 3], np.int32))
    A = torch.zeros(B, T, device="cuda")
    OL = torch.zeros(B, T, device="cuda")
    w = torch.full((B, T), 1.0 / 6, device="cuda")
    cfg = rlo.TrainConfig()
    with pytest.raises(rlo.InputError, match="missing old logprobs"):
        obj.ppo_gradient_fused(cfg, dev(torch, np.zeros((B, T), np.int32)), L, x, A, w)
    toks = np.zeros((B, T), np.int32)
    toks[1, 2] = V + 5
    obj.ppo_gradient_fused(cfg, dev(torch, toks), L, x, A, w, old_logprobs=OL)
    with pytest.raises(rlo.InputError, match=f"out-of-vocabulary token {V + 5}"):
        obj.sync()
    with pytest.raises((rlo.TrainingError, rlo.InputError)):
        obj.merge_gradients(cfg)  # the OOV row's NaN log-prob makes the loss non-finite


def test_fused_three_slices_in_flight(env, monkeypatch):
    """RLO_FUSED_NB=3 (gradient written two rows late) gives the same results."""
    torch, rlo, _ = env
    monkeypatch.setenv("RLO_FUSED_NB", "3")  # read when the handle is created
    obj = rlo.Objective(0)
    test_fused_matches_two_pass_and_oracle((torch, rlo, obj), "f32", "f32", 32000, 3, 1)
    test_fused_matches_two_pass_and_oracle((torch, rlo, obj), "f32", "bf16", 4099, 1, 3)
