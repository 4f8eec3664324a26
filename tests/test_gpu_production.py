"""The production kernels at the north_star's shapes, against the oracle.

Every vocab-pass instantiation the library ships (vocab.cu: one per dtype,
tensor count, mode and entropy flag) is reached here at the shape it is
selected for, through the C ABI (rlo_ppo_gradient / rlo_forward_logprobs /
rlo_objective_step_host_mb):

* bf16 V = 152064, P = 3 (BASELINE cfg 3-5): the long-row lockstep kernel
  (the three rows streamed together on a deferred offset, the FMA-pipe exp2
  on a quarter of the old/ref pairs) -- reduced-size
  end-to-end variants of cfg 3 (GRPO G=16, k3 0.001), cfg 4 (dual-clip c=3,
  global whitening, T = 16384, packed logits) and cfg 5 (GRPO G=8 + whitening),
  one full-size cfg 3 micro-batch through size-independent properties, the
  rows that defeat a lazy max / deferred offset: every element far below one
  spike that sits in a polynomial lane (the .y word of a uint4), actor rows
  whose later batches sit 5-40 nats above the first, -inf masked entries;
* bf16 P = 2: the same lockstep kernel with two tensors; both lockstep
  kernels at V = 32000 too, with old/ref rows far above and far below the
  actor's;
* bf16 P = 1 and forward_logprobs: two rows per warp in lockstep, each on its
  own deferred offset (a pair with an inactive or misaligned row: the
  lazy-running-max stream, mix 7);
* the fp32 and bf16 forward_logprobs instantiations with and without entropy.

Tolerance (north_star): |gpu - oracle| <= 1e-5 * max(1, |oracle|) for
log-probs, entropy and merged stats; 2e-5 for per-token loss / dlogp /
advantages (fp32 inputs); counts exact (clip counts within one token at an
fp32 rounding boundary).  Oracle = oracle/ (fp64, pinned to the reference)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5
QWEN_V = 152064


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2506_06122_b200 as rlo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, rlo, rlo.Objective(0)


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_close(got, want, tol=TOL, what=""):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
    assert np.all(err <= tol), f"{what}: max scaled err {err.max():.3g} at {np.argmax(err)}"


def close(g, r, tol=TOL):
    return abs(g - r) <= tol * max(1.0, abs(r))


def bf16_bits(torch, rows_f32):
    """float32 host rows -> (bf16 CUDA tensor, uint16 host bits for the oracle)."""
    t = torch.from_numpy(np.ascontiguousarray(rows_f32, dtype=np.float32)).to(torch.bfloat16)
    return t.cuda(), t.view(torch.int16).numpy().view(np.uint16)


def synth_models(torch, rlo, rows, V, seed, key_offset=0):
    """The bench's synthetic logits (include/rlo_synth.h) for actor/old/ref:
    device tensors and the oracle's host copies (same bits)."""
    dv, host = [], []
    for m in range(3):
        x = torch.empty(rows, V, dtype=torch.bfloat16, device="cuda")
        rlo.synth_logits(x, seed=seed, model=m, row_key_offset=key_offset)
        dv.append(x)
        host.append(np.stack([O.synth_row_raw(O.BF16, V, seed, m, key_offset + r) for r in range(rows)]))
    return dv, host


def valid_mask(B, T, lengths, mask=None):
    m = (np.arange(T)[None, :] < lengths[:, None]).ravel()
    return m if mask is None else m & (mask.ravel() != 0)


def run_objective(torch, rlo, obj, cfg, oc, B, T, V, lengths, tokens, logits_dev, logits_host, rewards_seq,
                  mask=None, seq_start=None, packed_rows=None):
    """compute_advantages -> ppo_gradient (P = 3) -> merge on the GPU, and the
    same through the oracle; asserts every per-token output and the stats."""
    L, K = dev(torch, lengths), dev(torch, tokens)
    M = None if mask is None else dev(torch, mask)
    adv = obj.compute_advantages(cfg, L, T=T, mask=M, scalar_rewards=dev(torch, rewards_seq))
    ss = None if seq_start is None else dev(torch, seq_start)
    outs = obj.ppo_gradient(cfg, K, L, logits_dev[0], adv, mask=M, old_logits=logits_dev[1],
                            ref_logits=logits_dev[2], seq_start=ss,
                            outputs=("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss"))
    st = obj.merge_gradients(cfg)
    o_adv, _ = O.compute_advantages(oc, B, T, lengths, mask, rewards_seq=rewards_seq.astype(np.float64))
    assert_close(adv.cpu().numpy().ravel(), o_adv, tol=2e-5, what="advantages")
    if seq_start is None:
        lps = [O.forward_logprobs(h, O.BF16, V, V, B, T, lengths, tokens) for h in logits_host]
    else:  # packed rows: the oracle walks each sequence's own rows
        lps = []
        for h in logits_host:
            lp, ent = np.zeros(B * T), np.zeros(B * T)
            for b in range(B):
                n = int(lengths[b])
                if n == 0:
                    continue
                rows = h[seq_start[b]:seq_start[b] + n]
                a, e, _ = O.forward_logprobs(rows, O.BF16, V, V, 1, n, np.array([n], np.int32), tokens[b, :n])
                lp[b * T:b * T + n], ent[b * T:b * T + n] = a, e
            lps.append((lp, ent))
    loss_tok, dlogp, part = O.ppo_loss(oc, B, T, lengths, mask, lps[0][0], lps[1][0], lps[2][0], o_adv, lps[0][1])
    want = O.merge(part[None], oc)
    m = valid_mask(B, T, lengths, mask)
    for name, k in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        assert_close(outs[name].cpu().numpy().ravel()[m], lps[k][0][m], what=name)
    assert_close(outs["entropy"].cpu().numpy().ravel()[m], lps[0][1][m], what="entropy")
    assert_close(outs["loss"].cpu().numpy().ravel(), loss_tok, tol=2e-5, what="loss_tok")
    assert_close(outs["dlogp"].cpu().numpy().ravel(), dlogp, tol=2e-5, what="dlogp")
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert close(getattr(st, k), want[k]), (k, getattr(st, k), want[k])
    for k in ("tokens", "seqs", "groups"):
        assert getattr(st, k) == want[k], k
    assert abs(st.clip_fraction - want["clip_fraction"]) * st.tokens <= 1
    assert abs(st.dual_clip_fraction - want["dual_clip_fraction"]) * st.tokens <= 1
    return st, want


# ---- reduced-size BASELINE cfg 3 / 4 / 5 through the production bf16 kernel ----------------------

def test_cfg3_reduced_default_kernel_vs_oracle(env):
    """cfg 3 (GRPO, 16 responses per prompt, k3 KL at 0.001, token-mean) on one
    group of 16 x 6 tokens at the Qwen vocabulary, bf16, P = 3."""
    torch, rlo, obj = env
    rng = np.random.default_rng(3)
    B, T, V, G = 16, 6, QWEN_V, 16
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    lengths[0] = T
    lg, host = synth_models(torch, rlo, B * T, V, seed=3)
    toks = torch.empty(B * T, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(toks, V, seed=3)  # drawn from the row's softmax, like sampled responses
    tokens = toks.cpu().numpy().reshape(B, T)
    tokens[1, :2] = rng.integers(0, V, 2)  # and two uniform tokens (low log-probs)
    rs = (rng.random(B) < 0.4).astype(np.float32)
    kw = dict(adv_estimator="grpo", group_size=G, kl_estimator="k3", kl_coef=0.001, loss_agg="token-mean")
    cfg = rlo.TrainConfig(**kw)
    oc = O.TrainConfig(adv_estimator=O.GRPO, group_size=G, kl_estimator=O.K3, kl_coef=0.001)
    run_objective(torch, rlo, obj, cfg, oc, B, T, V, lengths, tokens, lg, host, rs)


def test_cfg4_reduced_long_cot_packed_vs_oracle(env):
    """cfg 4 (long-CoT RLVR: dual-clip c = 3, global batch whitening, k3) with
    T = 16384 and packed (varlen) logits: one 2048-token response and seven
    short or empty ones in a group of 8."""
    torch, rlo, obj = env
    B, T, V, G = 8, 16384, QWEN_V, 8
    lengths = np.array([2048, 1, 2, 0, 5, 7, 3, 11], np.int32)
    seq_start = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    rows = int(lengths.sum())
    lg, host = synth_models(torch, rlo, rows, V, seed=4)
    tokens = np.zeros((B, T), np.int32)
    for b in range(B):
        for t in range(lengths[b]):
            tokens[b, t] = O.synth_token(4, seq_start[b] + t, V)
    rs = np.array([1, 0, 1, 1, 0, 0, 1, 0], np.float32)
    kw = dict(adv_estimator="grpo", group_size=G, whiten_advantages=True, dual_clip_c=3.0, kl_estimator="k3",
              kl_coef=0.001, loss_agg="token-mean")
    cfg = rlo.TrainConfig(**kw)
    oc = O.TrainConfig(adv_estimator=O.GRPO, group_size=G, whiten_advantages=1, dual_clip_c=3.0,
                       kl_estimator=O.K3, kl_coef=0.001)
    run_objective(torch, rlo, obj, cfg, oc, B, T, V, lengths, tokens, lg, host, rs, seq_start=seq_start)


def test_cfg5_reduced_grpo_whitened_vs_oracle(env):
    """cfg 5 (GRPO, 8 responses per prompt, global whitening) on two groups,
    with a response mask (agentic-style spans)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(5)
    B, T, V, G = 16, 5, QWEN_V, 8
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[3] = T
    mask = (rng.random((B, T)) < 0.8).astype(np.uint8)
    lg, host = synth_models(torch, rlo, B * T, V, seed=5, key_offset=1000)
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    rs = (rng.random(B) < 0.5).astype(np.float32)
    kw = dict(adv_estimator="grpo", group_size=G, whiten_advantages=True, kl_estimator="k3", kl_coef=0.001)
    cfg = rlo.TrainConfig(**kw)
    oc = O.TrainConfig(adv_estimator=O.GRPO, group_size=G, whiten_advantages=1, kl_estimator=O.K3, kl_coef=0.001)
    run_objective(torch, rlo, obj, cfg, oc, B, T, V, lengths, tokens, lg, host, rs, mask=mask)


def test_cfg3_full_micro_batch_properties(env):
    """One full cfg 3 micro-batch (16 x 2048 rows x 152064, three bf16 tensors,
    30 GB): sampled rows against the oracle, the whole micro-batch's reduction
    against the oracle applied to the GPU's own per-token values, and the
    ratio-one identity loss = -mean(A) (test_policy.cpp:339-355)."""
    torch, rlo, obj = env
    B, T, V, G = 16, 2048, QWEN_V, 16
    seed = 0
    L = []
    for m in range(3):
        x = torch.empty(B * T, V, dtype=torch.bfloat16, device="cuda")
        rlo.synth_logits(x, seed=seed, model=m)
        L.append(x)
    toks = torch.empty(B, T, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(toks, V, seed=seed)
    lengths = torch.full((B,), T, dtype=torch.int32, device="cuda")
    rs = torch.from_numpy((np.arange(B) % 3 == 0).astype(np.float32)).cuda()
    cfg = rlo.TrainConfig(adv_estimator="grpo", group_size=G, kl_estimator="k3", kl_coef=0.001)
    adv = obj.compute_advantages(cfg, lengths, T=T, scalar_rewards=rs)
    outs = obj.ppo_gradient(cfg, toks, lengths, L[0], adv, old_logits=L[1], ref_logits=L[2],
                            outputs=("logp", "old_logp", "ref_logp", "entropy"))
    st = obj.merge_gradients(cfg)
    rng = np.random.default_rng(33)
    tk = toks.cpu().numpy().ravel()
    for name, m in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        got = outs[name].cpu().numpy().ravel()
        for r in rng.choice(B * T, 12, replace=False):
            z = O.synth_row(O.BF16, V, seed, m, int(r))
            lse, ent = O.logsoftmax_row(z)
            assert close(got[r], z[tk[r]] - lse), (name, r)
            if m == 0:
                assert close(outs["entropy"].cpu().numpy().ravel()[r], ent), r
    lp, old, ref, ent = (outs[k].cpu().numpy().ravel().astype(np.float64)
                         for k in ("logp", "old_logp", "ref_logp", "entropy"))
    oc = O.TrainConfig(adv_estimator=O.GRPO, group_size=G, kl_estimator=O.K3, kl_coef=0.001)
    full = np.full(B, T, np.int32)
    o_adv, _ = O.compute_advantages(oc, B, T, full, rewards_seq=rs.cpu().numpy().astype(np.float64))
    assert_close(adv.cpu().numpy().ravel(), o_adv, tol=2e-5, what="adv")
    _, _, part = O.ppo_loss(oc, B, T, full, None, lp, old, ref, o_adv, ent)
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert close(getattr(st, k), want[k]), k
    assert st.tokens == B * T
    cfg1 = rlo.TrainConfig()
    obj.ppo_gradient(cfg1, toks, lengths, L[0], adv, old_logits=L[0])
    st1 = obj.merge_gradients(cfg1)
    # the old-policy row (no entropy) sends a quarter of its pairs through the
    # degree-4 FMA-pipe exp2 (<= 2.9e-6 per term), the actor row is all MUFU
    assert abs(st1.mean_ratio - 1.0) <= 2e-6 and close(st1.loss, -float(adv.double().mean()), 2e-6)


# ---- rows that defeat a lazy running max ---------------------------------------------------------

def spike_rows(V, spikes):
    """Rows of -1e4 (finite large-negative masking) with spikes; each spike
    sits in the .y word (elements 2..3 of 8) of its 16-byte vector -- the
    polynomial lane of the bf16 old/ref mix -- and past the first 8192
    elements, so the owning thread's running max is the -1e4 floor when the
    spike's chunk arrives and only a polynomial lane sees it."""
    rows = np.full((len(spikes), V), -1e4, np.float32)
    for i, sp in enumerate(spikes):
        for pos, val in sp:
            assert pos % 8 in (2, 3) and pos >= 8192
            rows[i, pos] = val
    return rows


SPIKES = [
    [(8194, 5.0)],                       # thread 0, second load batch
    [(8192 * 5 + 8 * 77 + 3, 50.0)],     # another thread and batch
    [(20000 * 8 // 8 + 2, 0.0), (150002, 7.0)],
    [(9000 * 8 + 2, -9000.0)],           # moderate offset (t ~ 1443, far above 127)
]


def test_bf16_spike_above_running_max_loss_pass(env):
    """old / ref rows of the P = 3 loss pass (lazy max + polynomial lanes): the
    spike dominates the lse; a wrapped 2^t would drop it."""
    torch, rlo, obj = env
    V = QWEN_V
    n = len(SPIKES)
    rows = spike_rows(V, SPIKES)
    actor = np.random.default_rng(1).standard_normal((n, V)).astype(np.float32) * 2
    da, ha = bf16_bits(torch, actor)
    dr, hr = bf16_bits(torch, rows)
    toks = np.array([[sp[0][0] for sp in SPIKES]], np.int32)
    lengths = np.array([n], np.int32)
    cfg = rlo.TrainConfig(kl_coef=0.001, kl_estimator="k3")
    outs = obj.ppo_gradient(cfg, dev(torch, toks), dev(torch, lengths), da, dev(torch, np.zeros((1, n), np.float32)),
                            old_logits=dr, ref_logits=dr, outputs=("logp", "old_logp", "ref_logp"))
    obj.merge_gradients(cfg)
    want = O.forward_logprobs(hr, O.BF16, V, V, 1, n, lengths, toks)[0]
    assert_close(outs["old_logp"].cpu().numpy().ravel(), want, what="old_logp (spike)")
    assert_close(outs["ref_logp"].cpu().numpy().ravel(), want, what="ref_logp (spike)")
    assert_close(outs["logp"].cpu().numpy().ravel(), O.forward_logprobs(ha, O.BF16, V, V, 1, n, lengths, toks)[0],
                 what="actor logp")


@pytest.mark.parametrize("entropy", [False, True])
def test_bf16_spike_above_running_max_forward_logprobs(env, entropy):
    """forward_logprobs at bf16 (no entropy: polynomial lanes; with entropy:
    all MUFU) on the same rows."""
    torch, rlo, obj = env
    V = QWEN_V
    n = len(SPIKES)
    dr, hr = bf16_bits(torch, spike_rows(V, SPIKES))
    toks = np.array([[sp[0][0] for sp in SPIKES]], np.int32)
    lengths = np.array([n], np.int32)
    out = obj.forward_logprobs(dr, dev(torch, toks), dev(torch, lengths), entropy=entropy)
    lp, ent, _ = O.forward_logprobs(hr, O.BF16, V, V, 1, n, lengths, toks)
    assert_close(out["logp"].cpu().numpy().ravel(), lp, what="logp (spike)")
    if entropy:
        assert_close(out["entropy"].cpu().numpy().ravel(), ent, what="entropy (spike)")


@pytest.mark.parametrize("V", [32000, QWEN_V])
@pytest.mark.parametrize("off_old,off_ref", [(200.0, -80.0), (30.0, -40.0), (-300.0, 120.0)])
def test_bf16_lockstep_offsets(env, off_old, off_ref, V):
    """bf16 P = 3 rows take the lockstep kernel on a deferred offset (any V),
    whose old/ref sums ride on the actor's offset: old/ref rows far above it (overflow side) or far
    below it (ex2.approx.ftz flushes the bulk of the row) must be redone with
    their own max."""
    torch, rlo, obj = env
    rng = np.random.default_rng(int(abs(off_old)))
    B, T = 4, 6
    lengths = np.array([6, 3, 5, 1], np.int32)
    base = rng.standard_normal((B * T, V)).astype(np.float32) * 2.5
    rows = [base, base + off_old + rng.standard_normal((B * T, V)).astype(np.float32) * 0.1,
            base + off_ref + rng.standard_normal((B * T, V)).astype(np.float32) * 0.1]
    pairs = [bf16_bits(torch, r) for r in rows]
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    adv = rng.uniform(-1, 1, (B, T)).astype(np.float32)
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3")
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), pairs[0][0], dev(torch, adv),
                            old_logits=pairs[1][0], ref_logits=pairs[2][0],
                            outputs=("logp", "old_logp", "ref_logp", "entropy"))
    obj.merge_gradients(cfg)
    m = valid_mask(B, T, lengths)
    for name, k in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        want, ent, _ = O.forward_logprobs(pairs[k][1], O.BF16, V, V, B, T, lengths, tokens)
        assert_close(outs[name].cpu().numpy().ravel()[m], want[m], what=f"{name} offset {off_old}/{off_ref}")
        if k == 0:
            assert_close(outs["entropy"].cpu().numpy().ravel()[m], ent[m], what="entropy")


LS_FIRST = 3 * 256 * 8  # elements in the long-row lockstep kernel's first batch (U = 3 vectors x 256 threads)


@pytest.mark.parametrize("pad", [0, 1])
@pytest.mark.parametrize("gap", [0.0, 5.0, 10.0, 14.0, 40.0, "spike", "masked", "shift250", "shift300", "shift-400"])
def test_bf16_long_lockstep_deferred_offset(env, gap, pad):
    """The long-row lockstep kernel (bf16, V = 152064, P = 3) sums every batch
    after a thread's first against that first batch's actor max.  Rows whose
    later elements sit `gap` nats above the first batch: below the redo cap
    (s < 2^32) the entropy's log2 s - w/s cancels the gap's bits and must stay
    within 1e-5; above it (gap 40, one +60 spike) the share is redone exactly;
    pad = 1: the same rows off 16-byte alignment (the per-tensor fallback);
    "masked": a third of the actor row is -inf (masked vocabulary: guarded
    redo); "shiftX": whole rows X nats off zero (the packed-bf16 clamp of the
    polynomial lanes holds for offsets below 256 nats, larger ones keep the
    fp32 clamp).  Old / ref rows carry the same shape shifted by +-25 nats."""
    torch, rlo, obj = env
    rng = np.random.default_rng(77 if isinstance(gap, str) else int(gap * 10))
    B, T, V = 2, 4, QWEN_V
    lengths = np.array([4, 3], np.int32)
    rows = rng.standard_normal((B * T, V)).astype(np.float32) * 1.5
    if gap == "spike":
        rows[:, LS_FIRST + 8 * 1000 + 5] = 60.0
    elif gap == "masked":
        rows[:, rng.choice(V, V // 3, replace=False)] = -np.inf
    elif isinstance(gap, str) and gap.startswith("shift"):
        rows += float(gap[5:])
    else:
        rows[:, LS_FIRST:] += gap
    tensors = [rows, rows[::-1] + 25.0, rows + rng.standard_normal(rows.shape).astype(np.float32) * 0.2 - 25.0]
    if gap == "masked":
        tensors[1] = np.where(np.isinf(rows), rows, tensors[1])
    pairs = [bf16_bits(torch, r) for r in tensors]
    if pad:  # a row stride of V + 1: rows off 16-byte alignment take the kernel's per-tensor deferred fallback
        for i, (d, h) in enumerate(pairs):
            full = torch.zeros(B * T, V + pad, dtype=torch.bfloat16, device="cuda")
            full[:, :V] = d
            pairs[i] = (full[:, :V], h)
    tokens = rng.integers(LS_FIRST, V, (B, T)).astype(np.int32)
    if gap == "masked":
        tokens = np.array([[int(np.argmax(r)) for r in rows]], np.int32).reshape(B, T)
    adv = rng.uniform(-1, 1, (B, T)).astype(np.float32)
    cfg = rlo.TrainConfig(kl_coef=0.001, kl_estimator="k3")
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), pairs[0][0], dev(torch, adv),
                            old_logits=pairs[1][0], ref_logits=pairs[2][0],
                            outputs=("logp", "old_logp", "ref_logp", "entropy"))
    obj.merge_gradients(cfg)
    m = valid_mask(B, T, lengths)
    for name, k in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        want, ent, _ = O.forward_logprobs(pairs[k][1], O.BF16, V, V, B, T, lengths, tokens)
        assert_close(outs[name].cpu().numpy().ravel()[m], want[m], what=f"{name} gap {gap}")
        if k == 0:
            assert_close(outs["entropy"].cpu().numpy().ravel()[m], ent[m], what=f"entropy gap {gap}")


@pytest.mark.parametrize("V", [QWEN_V, 32000])
@pytest.mark.parametrize("P", [1, 2])
def test_bf16_p1_p2_kernels(env, P, V):
    """bf16 loss pass with one or two logits tensors (old / ref log-probs
    precomputed) against the oracle: P = 1 takes the two-rows-per-warp kernel,
    P = 2 the lockstep kernel, both on deferred offsets; at V = 152064 the old rows of the first tokens are
    the spike rows that defeat a lazy max."""
    torch, rlo, obj = env
    rng = np.random.default_rng(90 + P)
    B, T = 2, 5
    lengths = np.array([5, 4], np.int32)
    lg, host = synth_models(torch, rlo, B * T, V, seed=11)
    old_rows = host[1].copy()
    old_dev = lg[1].clone()
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    if V == QWEN_V:
        sd, sh = bf16_bits(torch, spike_rows(V, SPIKES))
        old_dev[:len(SPIKES)] = sd
        old_rows[:len(SPIKES)] = sh
        tokens.ravel()[:len(SPIKES)] = [sp[0][0] for sp in SPIKES]  # finite ratios on the spike rows
    adv = rng.uniform(-1, 1, (B, T)).astype(np.float32)
    ref_in = rng.uniform(-12, -2, (B, T)).astype(np.float32)
    old_in = rng.uniform(-12, -2, (B, T)).astype(np.float32)
    cfg = rlo.TrainConfig(kl_coef=0.001, kl_estimator="k3")
    kw = dict(old_logits=old_dev) if P == 2 else dict(old_logprobs=dev(torch, old_in))
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), lg[0], dev(torch, adv),
                            ref_logprobs=dev(torch, ref_in), outputs=("logp", "old_logp", "entropy", "loss"), **kw)
    st = obj.merge_gradients(cfg)
    m = valid_mask(B, T, lengths)
    lp, ent, _ = O.forward_logprobs(host[0], O.BF16, V, V, B, T, lengths, tokens)
    old = O.forward_logprobs(old_rows, O.BF16, V, V, B, T, lengths, tokens)[0] if P == 2 else \
        old_in.astype(np.float64).ravel()
    assert_close(outs["logp"].cpu().numpy().ravel()[m], lp[m], what="logp")
    assert_close(outs["entropy"].cpu().numpy().ravel()[m], ent[m], what="entropy")
    assert_close(outs["old_logp"].cpu().numpy().ravel()[m], old[m], what="old_logp")
    oc = O.TrainConfig(kl_estimator=O.K3, kl_coef=0.001)
    loss_tok, _, part = O.ppo_loss(oc, B, T, lengths, None, lp, old, ref_in.astype(np.float64).ravel(),
                                   adv.astype(np.float64).ravel(), ent)
    assert_close(outs["loss"].cpu().numpy().ravel(), loss_tok, tol=2e-5, what="loss_tok")
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert close(getattr(st, k), want[k]), (k, getattr(st, k), want[k])


@pytest.mark.parametrize("pad", [8, 1, 16])
def test_bf16_row_alignments(env, pad):
    """The bf16 pass reads 32-byte pairs (LDG.256) when a row's aligned body
    starts on 32 bytes and 16-byte vectors otherwise: a row stride of V + 8
    alternates the two layouts row by row, V + 1 also shifts the scalar head,
    V + 16 keeps every row 32-byte aligned.  P = 3 loss pass and
    forward_logprobs against the oracle."""
    torch, rlo, obj = env
    rng = np.random.default_rng(100 + pad)
    B, T, V = 2, 3, QWEN_V
    lengths = np.array([3, 2], np.int32)
    rows = [rng.standard_normal((B * T, V)).astype(np.float32) * 3 for _ in range(3)]
    dev_rows, host_rows = [], []
    for r in rows:
        full = torch.zeros(B * T, V + pad, dtype=torch.bfloat16)
        full[:, :V] = torch.from_numpy(r).to(torch.bfloat16)
        dev_rows.append(full.cuda()[:, :V])
        host_rows.append(full[:, :V].contiguous().view(torch.int16).numpy().view(np.uint16))
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    K, L = dev(torch, tokens), dev(torch, lengths)
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k2")
    outs = obj.ppo_gradient(cfg, K, L, dev_rows[0], dev(torch, np.zeros((B, T), np.float32)),
                            old_logits=dev_rows[1], ref_logits=dev_rows[2],
                            outputs=("logp", "old_logp", "ref_logp", "entropy"))
    obj.merge_gradients(cfg)
    m = valid_mask(B, T, lengths)
    for name, k in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        want, ent, _ = O.forward_logprobs(host_rows[k], O.BF16, V, V, B, T, lengths, tokens)
        assert_close(outs[name].cpu().numpy().ravel()[m], want[m], what=f"{name} pad {pad}")
        if k == 0:
            assert_close(outs["entropy"].cpu().numpy().ravel()[m], ent[m], what="entropy")
    fl = obj.forward_logprobs(dev_rows[2], K, L, entropy=False)
    want, _, _ = O.forward_logprobs(host_rows[2], O.BF16, V, V, B, T, lengths, tokens)
    assert_close(fl["logp"].cpu().numpy().ravel()[m], want[m], what="forward_logprobs")


# ---- every shipped forward_logprobs instantiation --------------------------------------------------

@pytest.mark.parametrize("V,stride", [(100003, 100008), (70001, 70001), (65536, 65536), (65535, 65544)])
def test_bf16_long_rows_odd_vocab(env, V, stride):
    """bf16 rows in the lockstep kernel with a vocabulary that is not a
    multiple of the 16-byte vector: aligned rows (stride a multiple of 8) run
    the lockstep batches, the partial batch and the scalar tail; a contiguous
    odd vocabulary misaligns every other row (per-tensor fallback inside the
    same kernel).  P = 3 loss pass against the oracle."""
    torch, rlo, obj = env
    rng = np.random.default_rng(V)
    B, T = 2, 3
    lengths = np.array([3, 2], np.int32)
    dev_rows, host_rows = [], []
    for k in range(3):
        r = rng.standard_normal((B * T, V)).astype(np.float32) * 2.5 + (0.0, 9.0, -9.0)[k]
        full = torch.zeros(B * T, stride, dtype=torch.bfloat16)
        full[:, :V] = torch.from_numpy(r).to(torch.bfloat16)
        dev_rows.append(full.cuda()[:, :V])
        host_rows.append(full[:, :V].contiguous().view(torch.int16).numpy().view(np.uint16))
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    tokens[0, 0] = V - 1  # the scalar tail's last element
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3")
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), dev_rows[0],
                            dev(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32)),
                            old_logits=dev_rows[1], ref_logits=dev_rows[2],
                            outputs=("logp", "old_logp", "ref_logp", "entropy"))
    obj.merge_gradients(cfg)
    m = valid_mask(B, T, lengths)
    for name, k in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        want, ent, _ = O.forward_logprobs(host_rows[k], O.BF16, V, V, B, T, lengths, tokens)
        assert_close(outs[name].cpu().numpy().ravel()[m], want[m], what=f"{name} V {V} stride {stride}")
        if k == 0:
            assert_close(outs["entropy"].cpu().numpy().ravel()[m], ent[m], what="entropy")


@pytest.mark.parametrize("dt,V", [("f32", 32000), ("bf16", QWEN_V), ("bf16", 4096)])
@pytest.mark.parametrize("entropy", [False, True])
def test_forward_logprobs_instantiations(env, dt, V, entropy):
    torch, rlo, obj = env
    rng = np.random.default_rng(V + entropy)
    B, T = 3, 5
    lengths = np.array([5, 2, 4], np.int32)
    rows = rng.standard_normal((B * T, V)).astype(np.float32) * 3
    rows[np.arange(B * T), rng.integers(0, V, B * T)] += 9.0
    rows[2, ::5] = -np.inf  # masked vocabulary entries
    if dt == "bf16":
        x, host = bf16_bits(torch, rows)
        odt = O.BF16
    else:
        x, host, odt = dev(torch, rows), rows, O.F32
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    tokens[0, 2] = 1  # row 2 has -inf at multiples of 5: keep its token finite
    out = obj.forward_logprobs(x, dev(torch, tokens), dev(torch, lengths), entropy=entropy)
    lp, ent, _ = O.forward_logprobs(host, odt, V, V, B, T, lengths, tokens)
    m = valid_mask(B, T, lengths)
    assert_close(out["logp"].cpu().numpy().ravel()[m], lp[m], what="logp")
    assert not out["logp"].cpu().numpy().ravel()[~m].any()  # invalid positions are written as 0
    if entropy:
        assert_close(out["entropy"].cpu().numpy().ravel()[m], ent[m], what="entropy")


# ---- the first failing row in sample order ---------------------------------------------------------

def test_oov_reports_first_token_in_sample_order(env):
    """With many out-of-vocabulary tokens spread over many CTAs, the error names
    the first one in (sample, position) order, as the reference's loop does
    (policy.cpp:223-225) -- also across micro-batches (seq_offset)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(8)
    B, T, V = 64, 32, 512
    lengths = np.full(B, T, np.int32)
    lengths[5] = 3
    logits = dev(torch, rng.standard_normal((B * T, V)).astype(np.float32))
    for trial in range(3):
        tokens = rng.integers(0, V, (B, T)).astype(np.int32)
        bad = rng.choice(B * T, 40, replace=False)
        tokens.ravel()[bad] = V + rng.integers(0, 1000, 40)
        tokens[5, 10] = -77  # beyond length 3: not a response position, never reported
        valid = valid_mask(B, T, lengths)
        first = next(int(tokens.ravel()[r]) for r in range(B * T) if valid[r] and not 0 <= tokens.ravel()[r] < V)
        obj.forward_logprobs(logits, dev(torch, tokens), dev(torch, lengths))
        with pytest.raises(rlo.InputError) as e:
            obj.sync()
        assert str(e.value) == f"forward_logprobs: out-of-vocabulary token {first}", trial
    # loss pass over two micro-batches: the earlier micro-batch's OOV wins even
    # if the later one has an OOV at a smaller local row
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    tokens[40, 30] = V + 1   # micro-batch 0 (seqs 0..47), local row 40*T+30
    tokens[49, 0] = V + 2    # micro-batch 1 (seqs 48..63), local row 1*T+0
    adv = dev(torch, np.zeros((B, T), np.float32))
    cfg = rlo.TrainConfig()
    K, L = dev(torch, tokens), dev(torch, lengths)
    obj.ppo_gradient(cfg, K[48:], L[48:], logits[48 * T:], adv[48:], old_logits=logits[48 * T:], seq_offset=48)
    obj.ppo_gradient(cfg, K[:48], L[:48], logits[:48 * T], adv[:48], old_logits=logits[:48 * T], seq_offset=0)
    with pytest.raises(rlo.InputError) as e:
        obj.merge_gradients(cfg)
    assert str(e.value) == f"ppo_gradient: out-of-vocabulary token {V + 1}"


# ---- the micro-batched reference-facing call -------------------------------------------------------

def test_step_host_mb_equals_single_call(env):
    """rlo_objective_step_host_mb over micro-batches of 3 sequences gives the
    same advantages, log-probs and (bitwise) stats as one rlo_objective_step_host
    call over the whole batch; the callback sees the micro-batches in order."""
    torch, rlo, obj = env
    rng = np.random.default_rng(12)
    B, T, V, G = 12, 7, 4096, 4
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    rows = [rng.standard_normal((B * T, V)).astype(np.float32) * 2]
    rows += [rows[0] + rng.standard_normal((B * T, V)).astype(np.float32) * 0.1 for _ in range(2)]
    X = [dev(torch, r) for r in rows]
    rs = rng.integers(0, 2, B).astype(np.float32)
    cfg = rlo.TrainConfig(adv_estimator="grpo", group_size=G, whiten_advantages=True, kl_coef=0.01,
                          kl_estimator="k2")
    adv1, lp1 = np.zeros((B, T), np.float32), np.zeros((B, T), np.float32)
    st1 = obj.step_host(cfg, tokens, lengths, X[0], scalar_rewards=rs, old_logits=X[1], ref_logits=X[2],
                        adv_out=adv1, logp_out=lp1)
    seen = []

    def fn(i, b0, nb):
        seen.append((i, b0, nb))
        return X[0][b0 * T:(b0 + nb) * T], X[1][b0 * T:(b0 + nb) * T], X[2][b0 * T:(b0 + nb) * T]

    adv2, lp2 = np.zeros((B, T), np.float32), np.zeros((B, T), np.float32)
    st2 = obj.step_host_mb(cfg, tokens, lengths, 5, fn, scalar_rewards=rs, adv_out=adv2, logp_out=lp2)
    assert seen == [(0, 0, 5), (1, 5, 5), (2, 10, 2)]
    assert np.array_equal(adv1, adv2) and np.array_equal(lp1, lp2)
    for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl", "mean_entropy", "tokens"):
        assert getattr(st1, k) == getattr(st2, k), k

    def bad(i, b0, nb):
        if i == 1:
            raise ValueError("model forward failed")
        return fn(i, b0, nb)

    with pytest.raises(ValueError):
        obj.step_host_mb(cfg, tokens, lengths, 5, bad, scalar_rewards=rs)
    st3 = obj.step_host(cfg, tokens, lengths, X[0], scalar_rewards=rs, old_logits=X[1], ref_logits=X[2])
    assert st3.loss == st1.loss  # the aborted step left no partial accumulation behind


# ---- decode at tiny temperatures -----------------------------------------------------------------

@pytest.mark.parametrize("temp", [1e-6, 1e-7, 1e-8, 1e-9])
@pytest.mark.parametrize("scale", [20.0, 200.0])
def test_decode_tiny_temperature(env, temp, scale):
    """decode_next at T -> 0 is a greedy draw (the reference decodes at
    T = 1e-6, pipeline.cpp:539): tokens equal the fp64 oracle's for logits
    around 20..200, where an fp32 clamp bound formed in the logit domain broke
    exp's domain."""
    torch, rlo, obj = env
    rng = np.random.default_rng(int(scale))
    n, V = 16, 4099
    rows = (rng.standard_normal((n, V)) * 3 + scale).astype(np.float32)
    rows[: n // 2, 17] = rows[: n // 2].max(axis=1) + 1e-4 * scale  # a near-tie with the max
    rows[3, 5] = -np.inf
    x = dev(torch, rows)
    keys = rng.integers(0, 2**62, n).astype(np.int64)
    pos = rng.integers(0, 1000, n).astype(np.int64)
    tok, lp = obj.decode_sample(x, temp, 7, 2, dev(torch, keys), dev(torch, pos))
    tok, lp = tok.cpu().numpy(), lp.cpu().numpy()
    for i in range(n):
        want, want_lp = O.decode_next(rows[i].astype(np.float64), temp, 7, 2, int(keys[i]), int(pos[i]))
        assert tok[i] == want, (i, tok[i], want)
        assert tok[i] == int(np.argmax(rows[i]))  # greedy at this temperature (no exact ties here)
        assert abs(lp[i] - want_lp) <= 1e-5 * max(1.0, abs(want_lp))


# ---- NaN logits propagate (policy.cpp:117-121: the log-sum-exp of a row holding a NaN is NaN) ------

@pytest.mark.parametrize("dt,V", [("bf16", QWEN_V), ("bf16", 32000), ("f32", 32000)])
def test_nan_logit_propagates_loss_pass(env, dt, V):
    """A NaN in one row of each tensor -- in a MUFU lane (actor) and in the
    polynomial lanes (.y word, old / ref) past the first batch -- makes that
    token's log-prob NaN (no clamp turns it into a finite term, no redo hides
    it); the other tokens stay finite and the merge refuses the step like the
    reference (TrainingError, policy.cpp:441-448)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(5)
    B, T = 1, 4
    lengths = np.array([4], np.int32)
    rows = [rng.standard_normal((B * T, V)).astype(np.float32) * 2 for _ in range(3)]
    rows[0][0, 8200] = np.nan   # actor, row 0
    rows[1][1, 8194] = np.nan   # old, row 1 (polynomial lane)
    rows[2][2, 20003] = np.nan  # ref, row 2 (polynomial lane)
    if dt == "bf16":
        x = [bf16_bits(torch, r)[0] for r in rows]
    else:
        x = [dev(torch, r) for r in rows]
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3")
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), x[0], dev(torch, np.zeros((B, T), np.float32)),
                            old_logits=x[1], ref_logits=x[2], outputs=("logp", "old_logp", "ref_logp", "entropy"))
    with pytest.raises(rlo.TrainingError):
        obj.merge_gradients(cfg)
    lp, old, ref = (outs[k].cpu().numpy().ravel() for k in ("logp", "old_logp", "ref_logp"))
    assert np.isnan(lp[0]) and np.isnan(outs["entropy"].cpu().numpy().ravel()[0])
    assert np.isnan(old[1]) and np.isnan(ref[2])
    assert np.isfinite(lp[1:]).all() and np.isfinite(old[[0, 2, 3]]).all() and np.isfinite(ref[[0, 1, 3]]).all()


@pytest.mark.parametrize("dt,V", [("bf16", QWEN_V), ("f32", 32000)])
@pytest.mark.parametrize("entropy", [False, True])
def test_nan_logit_propagates_forward_logprobs(env, dt, V, entropy):
    torch, rlo, obj = env
    rng = np.random.default_rng(6)
    rows = rng.standard_normal((3, V)).astype(np.float32) * 2
    rows[1, 8194] = np.nan  # polynomial lane of the no-entropy bf16 mix
    x = bf16_bits(torch, rows)[0] if dt == "bf16" else dev(torch, rows)
    out = obj.forward_logprobs(x, dev(torch, np.array([[5, 6, 7]], np.int32)), dev(torch, np.array([3], np.int32)),
                               entropy=entropy)
    lp = out["logp"].cpu().numpy().ravel()
    assert np.isnan(lp[1]) and np.isfinite(lp[[0, 2]]).all()
    if entropy:
        assert np.isnan(out["entropy"].cpu().numpy().ravel()[1])
