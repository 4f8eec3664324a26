"""GPU edge cases the reference's contracts imply: degenerate shapes, masked /
infinite logits, extreme magnitudes, padded row strides with garbage, bad
lengths, out-of-order micro-batches.  Oracle = oracle/ (fp64)."""
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


def close(g, r, tol=1e-5):
    return abs(g - r) <= tol * max(1.0, abs(r))


def test_vocab_of_one(env):
    torch, rlo, obj = env
    x = dev(torch, np.array([[3.5], [-2.0]], np.float32))
    out = obj.forward_logprobs(x, dev(torch, np.zeros((1, 2), np.int32)), dev(torch, np.array([2], np.int32)),
                               entropy=True)
    assert out["logp"].abs().max().item() < 1e-6 and out["entropy"].abs().max().item() < 1e-6


@pytest.mark.parametrize("V", [64, 4096, 32000])
def test_minus_inf_logits_and_extremes(env, V):
    torch, rlo, obj = env
    rng = np.random.default_rng(V)
    rows = rng.standard_normal((6, V)).astype(np.float32) * 3
    rows[0, rng.integers(0, V, V // 4)] = -np.inf   # masked vocabulary entries
    rows[1] *= 1000.0                               # |z| ~ 3e3: max subtraction must keep exp finite
    rows[2] = 1e-3 * rows[2]                        # near-uniform
    rows[3, : V // 2] = -np.inf                     # half the row masked
    rows[4] -= 1e4                                  # large negative offset
    rows[5, 7] = 80.0                               # one dominant logit
    toks = np.array([[int(np.argmax(r)) for r in rows]], np.int32)
    out = obj.forward_logprobs(dev(torch, rows), dev(torch, toks), dev(torch, np.array([6], np.int32)), entropy=True)
    lp, ent = out["logp"].cpu().numpy().ravel(), out["entropy"].cpu().numpy().ravel()
    for i in range(6):
        lse, h = O.logsoftmax_row(rows[i].astype(np.float64))
        assert close(lp[i], float(rows[i, toks[0, i]]) - lse), (i, lp[i])  # fp64: a float32 difference rounds lse
        assert np.isfinite(ent[i]) and abs(ent[i] - h) <= 2e-5 * max(1.0, h), (i, ent[i], h)


def test_padded_stride_garbage_is_never_read(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(1)
    V, S, B, T = 1000, 1024, 3, 5
    buf = np.full((B * T, S), np.nan, np.float32)   # NaN in the padding columns
    buf[:, :V] = rng.standard_normal((B * T, V)).astype(np.float32)
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    x = dev(torch, buf)[:, :V]
    out = obj.forward_logprobs(x, dev(torch, toks), dev(torch, np.array([5, 3, 0], np.int32)), entropy=True)
    lp, ent, _ = O.forward_logprobs(buf, O.F32, V, S, B, T, [5, 3, 0], toks)
    got = out["logp"].cpu().numpy().ravel()
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got - lp)) < 2e-5


def test_bad_length_is_input_error(env):
    torch, rlo, obj = env
    x = dev(torch, np.zeros((8, 16), np.float32))
    obj.forward_logprobs(x, dev(torch, np.zeros((2, 4), np.int32)), dev(torch, np.array([4, 9], np.int32)))
    with pytest.raises(rlo.InputError, match="sample '1'.*outside"):
        obj.sync()


def test_empty_shapes_are_noops(env):
    torch, rlo, obj = env
    cfg = rlo.TrainConfig()
    x = torch.zeros(0, 16, device="cuda")
    out = obj.forward_logprobs(x, torch.zeros(0, 4, dtype=torch.int32, device="cuda"),
                               torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert out["logp"].numel() == 0
    obj.ppo_gradient(cfg, torch.zeros(0, 4, dtype=torch.int32, device="cuda"),
                     torch.zeros(0, dtype=torch.int32, device="cuda"), x, torch.zeros(0, 4, device="cuda"),
                     old_logprobs=torch.zeros(0, 4, device="cuda"))
    with pytest.raises(rlo.TrainingError, match="no loss-participating tokens"):
        obj.merge_gradients(cfg)


def test_out_of_order_micro_batches(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(8)
    B, T, V = 9, 7, 2048
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    x = torch.randn(B * T, V, device="cuda") * 2
    adv = dev(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32))
    old = dev(torch, rng.uniform(-9, -6, (B, T)).astype(np.float32))
    cfg = rlo.TrainConfig(loss_agg="group-mean", group_size=3)
    L, K = dev(torch, lengths), dev(torch, toks)
    obj.ppo_gradient(cfg, K, L, x, adv, old_logprobs=old)
    st1, p1 = obj.merge_gradients(cfg, with_partials=True)
    for s0 in (6, 0, 3):  # reverse order of whole groups
        rs = slice(s0 * T, (s0 + 3) * T)
        obj.ppo_gradient(cfg, K[s0:s0 + 3], L[s0:s0 + 3], x[rs], adv[s0:s0 + 3], old_logprobs=old[s0:s0 + 3],
                         seq_offset=s0)
    st2, p2 = obj.merge_gradients(cfg, with_partials=True)
    assert np.array_equal(p1, p2) and st1 == st2


def test_all_masked_batch_raises_reference_error(env):
    torch, rlo, obj = env
    cfg = rlo.TrainConfig()
    B, T = 2, 3
    obj.ppo_gradient(cfg, dev(torch, np.zeros((B, T), np.int32)), dev(torch, np.array([3, 2], np.int32)),
                     torch.zeros(B * T, 8, device="cuda"), torch.zeros(B, T, device="cuda"),
                     mask=torch.zeros(B, T, dtype=torch.uint8, device="cuda"), old_logprobs=torch.zeros(B, T, device="cuda"))
    with pytest.raises(rlo.TrainingError) as e:
        obj.merge_gradients(cfg)
    assert str(e.value) == "merge_gradients: batch contains no loss-participating tokens"


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_unaligned_rows_head_body_tail(env, dt):
    """V = 50257 in a contiguous tensor: every row starts at a different
    offset from a 16-byte boundary (scalar head, vector body, scalar tail)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(7)
    B, T, V = 3, 11, 50257
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    x = (torch.randn(B * T, V, generator=torch.Generator().manual_seed(3)) * 3).to(tdt).cuda()
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    toks[0, :8] = np.arange(8)  # tokens inside the scalar head
    out = obj.forward_logprobs(x, dev(torch, toks), dev(torch, np.full(B, T, np.int32)), entropy=True)
    lp, ent = out["logp"].cpu().numpy().ravel(), out["entropy"].cpu().numpy().ravel()
    rows = x.float().cpu().numpy().astype(np.float64)
    for i in range(B * T):
        lse, h = O.logsoftmax_row(rows[i])
        assert close(lp[i], rows[i, toks.ravel()[i]] - lse), i
        assert abs(ent[i] - h) <= 2e-5 * max(1.0, h), i
    # backward epilogue on the same unaligned rows (fp32 gradient) vs the oracle
    w = torch.full((B, T), 0.5, device="cuda")
    dl = torch.full((B, T), -1.25, device="cuda")
    lse = torch.from_numpy(np.array([O.logsoftmax_row(r)[0] for r in rows], np.float32).reshape(B, T)).cuda()
    g = obj.logits_backward(dev(torch, toks), dev(torch, np.full(B, T, np.int32)), x, lse, dl, w,
                            grad_dtype=torch.float32).cpu().numpy()
    for i in (0, 1, 17, B * T - 1):
        want = O.logits_backward_row(rows[i], int(toks.ravel()[i]), 0.5 * -1.25)
        assert np.abs(g[i] - want).max() <= 1e-5 * 0.625 + 1e-12, i


def test_backward_with_fp64_lse_at_extreme_offsets(env):
    """Rows offset by +-1e4: the two-pass backward rebuilt from the fp64 lse
    (rlo_token_out.lse64 -> rlo_logits_backward64) matches the oracle's
    gradient to 1e-5; the fp32 lse carries its own rounding (ulp(1e4)/2)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(12)
    B, T, V = 2, 3, 4096
    rows = (rng.standard_normal((B * T, V)) * 3).astype(np.float32)
    rows[::2] -= 1e4
    rows[1::2] += 1e4
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    L = dev(torch, np.array([T, T], np.int32))
    x = dev(torch, rows)
    cfg = rlo.TrainConfig()
    old = dev(torch, np.full((B, T), -7.0, np.float32))
    outs = obj.ppo_gradient(cfg, dev(torch, toks), L, x, dev(torch, np.ones((B, T), np.float32)), old_logprobs=old,
                            outputs=("dlogp", "lse", "lse64"))
    obj.merge_gradients(cfg)
    w = torch.full((B, T), 0.25, device="cuda")
    g64 = obj.logits_backward(dev(torch, toks), L, x, outs["lse64"], outs["dlogp"], w, grad_dtype=torch.float32)
    G = g64.cpu().numpy()
    dl = outs["dlogp"].cpu().numpy().ravel()
    for i in range(B * T):
        scale = float(np.float32(0.25) * np.float32(dl[i]))
        want = O.logits_backward_row(rows[i].astype(np.float64), int(toks.ravel()[i]), scale)
        assert np.abs(G[i] - want).max() <= 1e-5 * abs(scale) + 1e-12, (i, np.abs(G[i] - want).max())
    assert abs(float(outs["lse64"][0, 0]) - O.logsoftmax_row(rows[0].astype(np.float64))[0]) <= 1e-6 * 1e4
