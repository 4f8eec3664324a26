"""Packed (varlen) logits layout: rlo_logits.seq_start maps token (b, t) to
row seq_start[b] + t of a [sum(lengths), V] tensor (padded
[B,T] or packed with cu_seqlens).  Every entry point must give the padded
layout's results — bit-identical when rows are 16-byte aligned (the same
element-to-thread split), within fp32 rounding otherwise (a row's scalar head
depends on its address) — read no padding rows, and write gradient rows only
for tokens that exist."""
import numpy as np
import pytest

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


def _ragged(torch, seed, B, T, V, dt, P):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[0] = T
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    gen = torch.Generator().manual_seed(seed)
    pad = [(torch.randn(B * T, V, generator=gen) * 3).to(tdt) for _ in range(P)]
    valid = np.concatenate([np.arange(b * T, b * T + lengths[b]) for b in range(B)])
    for x in pad:  # padding rows hold NaN: any read of them would poison the results
        inval = np.setdiff1d(np.arange(B * T), valid)
        x[torch.from_numpy(inval)] = float("nan")
    packed = [x[torch.from_numpy(valid)].contiguous().cuda() for x in pad]
    pad = [x.cuda() for x in pad]
    start = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    mask = (rng.random((B, T)) < 0.85).astype(np.uint8)
    adv = rng.uniform(-1.5, 1.5, (B, T)).astype(np.float32)
    return lengths, pad, packed, dev(torch, start), valid, toks, mask, adv


@pytest.mark.parametrize("dt,V,P", [("f32", 4099, 3), ("bf16", 2048, 2), ("f32", 32000, 1)])
def test_packed_equals_padded(env, dt, V, P):
    torch, rlo, obj = env
    B, T = 6, 9
    lengths, pad, packed, start, valid, toks, mask, adv = _ragged(torch, V + P, B, T, V, dt, P)
    L, K, M, A = dev(torch, lengths), dev(torch, toks), dev(torch, mask), dev(torch, adv)
    old = dev(torch, np.full((B, T), -7.0, np.float32))
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3", loss_agg="seq-mean-token-mean")
    # forward_logprobs (all valid positions)
    exact = (V * (4 if dt == "f32" else 2)) % 16 == 0

    def same(x, y, what):
        if exact:
            assert torch.equal(x, y), what
        else:
            assert torch.allclose(x, y, rtol=2e-6, atol=1e-7), what
    f1 = obj.forward_logprobs(pad[0], K, L, entropy=True, token_logit=True)
    f2 = obj.forward_logprobs(packed[0], K, L, entropy=True, token_logit=True, seq_start=start)
    for k in f1:
        same(f1[k], f2[k], k)

    def kw(x):
        d = {"old_logits": x[1]} if P >= 2 else {"old_logprobs": old}
        if P >= 3:
            d["ref_logits"] = x[2]
        else:
            d["ref_logprobs"] = old
        return d
    outs = ("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss", "lse")
    o1 = obj.ppo_gradient(cfg, K, L, pad[0], A, mask=M, outputs=outs, **kw(pad))
    s1 = obj.merge_gradients(cfg)
    o2 = obj.ppo_gradient(cfg, K, L, packed[0], A, mask=M, outputs=outs, seq_start=start, **kw(packed))
    s2 = obj.merge_gradients(cfg)
    if exact:
        assert s1 == s2
    else:
        assert s1.tokens == s2.tokens and abs(s1.loss - s2.loss) <= 1e-6 * max(1.0, abs(s1.loss))
    for k in outs:
        same(o1[k], o2[k], k)
    # backward epilogue and the fused update pass: gradient rows exist only for real tokens
    cnt = obj.batch_counts(cfg, L, T, mask=M)
    w = obj.loss_weights(cfg, L, cnt, T, mask=M)
    g1 = obj.logits_backward(K, L, pad[0], o1["lse"], o1["dlogp"], w, grad_dtype=torch.float32)
    n = len(valid)
    sentinel = 12345.0
    g2 = torch.full((n + 3, V), sentinel, device="cuda")
    obj.logits_backward(K, L, packed[0], o2["lse"], o2["dlogp"], w, grad=g2[:n], seq_start=start)
    same(g1[torch.from_numpy(valid).cuda()], g2[:n], "backward")
    assert bool((g2[n:] == sentinel).all())
    _, f1g = obj.ppo_gradient_fused(cfg, K, L, pad[0], A, w, mask=M, grad_dtype=torch.float32, **kw(pad))
    obj.merge_gradients(cfg)
    g3 = torch.full((n + 3, V), sentinel, device="cuda")
    obj.ppo_gradient_fused(cfg, K, L, packed[0], A, w, mask=M, grad=g3[:n], seq_start=start, **kw(packed))
    obj.merge_gradients(cfg)
    same(f1g[torch.from_numpy(valid).cuda()], g3[:n], "fused")
    assert bool((g3[n:] == sentinel).all())
