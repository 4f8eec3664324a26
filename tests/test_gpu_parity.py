"""GPU parity tests: the sm_100a path through the C ABI (librlo.so) against
the golden fixtures produced by the reference's own code and against the CPU
oracle.  Tolerance (north_star): |gpu - ref| <= 1e-5 * max(1, |ref|) for
floating point; bit-exact for token gathers, masks, counts and the synthetic
generator."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-5


def golden(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


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


# ---- synthetic generator (bench inputs) --------------------------------------

def test_synth_generator_bit_exact(env):
    torch, rlo, _ = env
    for dtype, V, tdt in [(O.F32, 32000, torch.float32), (O.BF16, 152064, torch.bfloat16), (O.F32, 1001, torch.float32)]:
        x = torch.empty(3, V, dtype=tdt, device="cuda")
        for model in (0, 1, 2):
            rlo.synth_logits(x, seed=7, model=model, row_key_offset=11)
            got = x.view(torch.int32 if tdt == torch.float32 else torch.int16).cpu().numpy()
            for r in range(3):
                want = O.synth_row_raw(dtype, V, 7, model, 11 + r).view(np.int32 if dtype == O.F32 else np.int16)
                assert np.array_equal(got[r], want)
    toks = torch.empty(1000, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(toks, 152064, seed=3, row_key_offset=5, key_rows=300)
    want = [O.synth_token(3, (5 + i) % 300, 152064) for i in range(1000)]
    assert toks.cpu().numpy().tolist() == want


# ---- forward_logprobs ---------------------------------------------------------

def test_forward_logprobs_matches_reference_rows(env):
    torch, rlo, obj = env
    d = np.load(os.path.join(G, "logsoftmax.npz"))
    for off, V, tok, ref_lp in zip(d["offsets"], d["V"], d["tokens"], d["ref_lp"]):
        row = d["rows"][off:off + V].astype(np.float32)
        for stride in (V, V + (-V) % 4 + 4):  # unaligned (scalar path) and 16B-aligned padded rows
            buf = np.zeros((1, stride), np.float32)
            buf[0, :V] = row
            t = dev(torch, buf)[:, :V]
            out = obj.forward_logprobs(t, dev(torch, np.array([[tok]], np.int32)), dev(torch, np.array([1], np.int32)),
                                       entropy=True, token_logit=True)
            assert close(out["logp"].item(), ref_lp), (V, stride)
            assert out["token_logit"].item() == row[tok]  # bit-exact gather
            _, ent = O.logsoftmax_row(row.astype(np.float64))
            assert close(out["entropy"].item(), ent)


def test_forward_logprobs_synthetic_batches(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(1)
    for dtype, V, tdt in [(O.F32, 32000, torch.float32), (O.BF16, 152064, torch.bfloat16), (O.BF16, 4096, torch.bfloat16)]:
        B, T = 5, 7
        lengths = rng.integers(0, T + 1, B).astype(np.int32)
        lengths[0] = T
        x = torch.empty(B * T, V, dtype=tdt, device="cuda")
        rlo.synth_logits(x, seed=5, model=1)
        toks = torch.empty(B * T, dtype=torch.int32, device="cuda")
        rlo.synth_tokens(toks, V, seed=5)
        out = obj.forward_logprobs(x, toks.view(B, T), dev(torch, lengths), entropy=True)
        rows = np.stack([O.synth_row_raw(dtype, V, 5, 1, r) for r in range(B * T)])
        lp, ent, _ = O.forward_logprobs(rows, dtype, V, V, B, T, lengths, toks.cpu().numpy())
        assert_close(out["logp"].cpu().numpy().ravel(), lp, what="logp")
        assert_close(out["entropy"].cpu().numpy().ravel(), ent, what="entropy")


def test_forward_logprobs_oov_is_input_error(env):
    torch, rlo, obj = env
    d = np.load(os.path.join(G, "forward_logprobs.npz"))
    row, lengths = d["row"], d["lengths"]
    B, T, V = len(lengths), len(d["tokens"]) // len(lengths), row.size
    logits = dev(torch, np.tile(row, (B * T, 1)))
    out = obj.forward_logprobs(logits, dev(torch, d["tokens"].reshape(B, T)), dev(torch, lengths))
    obj.sync()
    assert_close(out["logp"].cpu().numpy().ravel(), d["ref_lp"], what="forward_logprobs batch")
    code, msg = golden("misc.json")["oov_error"]
    obj.forward_logprobs(logits, dev(torch, d["bad_tokens"].reshape(B, T)), dev(torch, lengths))
    with pytest.raises(rlo.InputError) as e:
        obj.sync()
    assert str(e.value) == msg
    obj.sync()  # error state is cleared


# ---- advantages -----------------------------------------------------------------

def _arr(x, dt=np.float32):
    return None if x is None else np.asarray(x, dtype=dt)


def test_advantages_match_reference(env):
    torch, rlo, obj = env
    for c in golden("advantages.json")["cases"]:
        cfg = rlo.TrainConfig(**c["cfg"])
        B, T = c["B"], c["T"]
        kw = dict(T=T, mask=None if c["mask"] is None else dev(torch, _arr(c["mask"], np.uint8).reshape(B, T)),
                  rewards=None if c["rewards_tok"] is None else dev(torch, _arr(c["rewards_tok"]).reshape(B, T)),
                  scalar_rewards=None if c["rewards_seq"] is None else dev(torch, _arr(c["rewards_seq"])))
        lengths = dev(torch, _arr(c["lengths"], np.int32))
        if c["error"]:
            with pytest.raises(rlo.InputError) as e:
                obj.compute_advantages(cfg, lengths, **kw)
            assert str(e.value) == c["error"][1]
            continue
        adv = obj.compute_advantages(cfg, lengths, **kw)
        # fp32 inputs: compare against the oracle on the same fp32 inputs and against the reference (fp64 inputs)
        assert_close(adv.cpu().numpy().ravel(), c["ref_adv"], tol=2e-5, what=c["name"])


@pytest.mark.parametrize("est", ["reinforce", "gae", "grpo"])
@pytest.mark.parametrize("whiten", [False, True])
def test_advantages_vs_oracle(env, est, whiten):
    torch, rlo, obj = env
    rng = np.random.default_rng([("reinforce", "gae", "grpo").index(est), int(whiten)])
    for B, T in [(16, 40), (8, 5000), (4, 1)]:
        G = 4
        lengths = rng.integers(0, T + 1, B).astype(np.int32)
        lengths[1] = T
        mask = (rng.random((B, T)) < 0.8).astype(np.uint8)
        rt = (rng.standard_normal((B, T)) * 0.3).astype(np.float32)
        rt[0, 0] = 50.0
        rs = rng.integers(0, 2, B).astype(np.float32)
        vals = (rng.standard_normal((B, T)) * 0.5).astype(np.float32)
        kw = dict(adv_estimator=est, gamma=0.99 if est != "grpo" else 1.0, lambd=0.95, whiten_advantages=whiten,
                  group_size=G, advantage_clip=3.0)
        cfg = rlo.TrainConfig(**kw)
        oc = O.TrainConfig(**{**kw, "adv_estimator": {"reinforce": 0, "grpo": 1, "gae": 2}[est]})
        use_tok = est != "grpo"
        adv, ret = obj.compute_advantages(cfg, dev(torch, lengths), T=T, mask=dev(torch, mask),
                                          rewards=dev(torch, rt) if use_tok else None,
                                          scalar_rewards=None if use_tok else dev(torch, rs),
                                          values=dev(torch, vals) if est == "gae" else None, returns=True)
        o_adv, o_ret = O.compute_advantages(oc, B, T, lengths, mask, rt.astype(np.float64) if use_tok else None,
                                            None if use_tok else rs.astype(np.float64),
                                            vals.astype(np.float64) if est == "gae" else None)
        assert_close(adv.cpu().numpy().ravel(), o_adv, tol=2e-5, what=f"{est} adv B={B} T={T}")
        assert_close(ret.cpu().numpy().ravel(), o_ret, tol=2e-5, what=f"{est} returns")


# ---- loss ---------------------------------------------------------------------

def test_ppo_stats_match_reference_b2(env):
    torch, rlo, obj = env
    for c in golden("ppo_stats.json")["cases"]:
        B, T, V = c["B"], c["T"], c["V"]
        cfg = rlo.TrainConfig(**c["cfg"])
        row = np.asarray(c["row"], np.float32)
        logits = dev(torch, np.tile(row, (B * T, 1)))
        mask = None if c["mask"] is None else dev(torch, _arr(c["mask"], np.uint8).reshape(B, T))
        ref = None if c["ref"] is None else dev(torch, _arr(c["ref"]).reshape(B, T))
        obj.ppo_gradient(cfg, dev(torch, _arr(c["tokens"], np.int32).reshape(B, T)),
                         dev(torch, _arr(c["lengths"], np.int32)), logits, dev(torch, _arr(c["adv"]).reshape(B, T)),
                         mask=mask, old_logprobs=dev(torch, _arr(c["old"]).reshape(B, T)), ref_logprobs=ref)
        st = obj.merge_gradients(cfg)
        want = c["ref_stats"]
        for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl"):
            assert close(getattr(st, k), want[k], tol=2e-5), (k, getattr(st, k), want[k])
        assert st.tokens == want["tokens"]


def _random_case(rng, B, T, V, dtype, masked=True):
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    lengths[0] = T
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    mask = (rng.random((B, T)) < 0.85).astype(np.uint8) if masked else None
    adv = rng.uniform(-2, 2, (B, T)).astype(np.float32)
    rows = [rng.standard_normal((B * T, V)).astype(np.float32) * 2.5]
    rows.append(rows[0] + rng.standard_normal((B * T, V)).astype(np.float32) * 0.15)
    rows.append(rows[0] + rng.standard_normal((B * T, V)).astype(np.float32) * 0.15)
    if dtype == O.BF16:
        import torch
        rows = [torch.from_numpy(r).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16) for r in rows]
    return lengths, tokens, mask, adv, rows


def _dev_logits(torch, r, dtype):
    t = dev(torch, r.view(np.int16) if dtype == O.BF16 else r)
    return t.view(torch.bfloat16) if dtype == O.BF16 else t


@pytest.mark.parametrize("dtype", [O.F32, O.BF16])
@pytest.mark.parametrize("agg", [0, 1, 2, 3])
@pytest.mark.parametrize("kl_est", [0, 1, 2])
def test_fused_loss_vs_oracle(env, dtype, agg, kl_est):
    torch, rlo, obj = env
    rng = np.random.default_rng(100 * dtype + 10 * agg + kl_est)
    B, T, V = 8, 12, 2048 + 8 * (agg + 1)
    lengths, tokens, mask, adv, rows = _random_case(rng, B, T, V, dtype)
    kw = dict(clip_eps=0.2, kl_coef=0.05, kl_estimator=kl_est, loss_agg=agg, group_size=4,
              dual_clip_c=3.0 if agg % 2 else 0.0)
    cfg = rlo.TrainConfig(**kw)
    outs = obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), _dev_logits(torch, rows[0], dtype),
                            dev(torch, adv), mask=dev(torch, mask), old_logits=_dev_logits(torch, rows[1], dtype),
                            ref_logits=_dev_logits(torch, rows[2], dtype),
                            outputs=("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss"))
    st = obj.merge_gradients(cfg)
    lps = [O.forward_logprobs(r, dtype, V, V, B, T, lengths, tokens) for r in rows]
    oc = O.TrainConfig(**kw)
    loss_tok, dlogp, part = O.ppo_loss(oc, B, T, lengths, mask, lps[0][0], lps[1][0], lps[2][0], adv, lps[0][1])
    want = O.merge(part[None], oc)
    m = (mask.ravel() != 0) & (np.arange(T)[None, :] < lengths[:, None]).ravel()
    assert_close(outs["logp"].cpu().numpy().ravel()[m], lps[0][0][m], what="logp")
    assert_close(outs["old_logp"].cpu().numpy().ravel()[m], lps[1][0][m], what="old_logp")
    assert_close(outs["ref_logp"].cpu().numpy().ravel()[m], lps[2][0][m], what="ref_logp")
    assert_close(outs["entropy"].cpu().numpy().ravel()[m], lps[0][1][m], what="entropy")
    assert_close(outs["loss"].cpu().numpy().ravel(), loss_tok, tol=2e-5, what="loss_tok")
    assert_close(outs["dlogp"].cpu().numpy().ravel(), dlogp, tol=2e-5, what="dlogp")
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert close(getattr(st, k), want[k]), (k, getattr(st, k), want[k])
    for k in ("tokens", "seqs", "groups"):
        assert getattr(st, k) == want[k]
    # counts are exact unless a ratio sits within fp32 rounding of a clip boundary
    assert abs(st.clip_fraction - want["clip_fraction"]) * st.tokens <= 1
    assert abs(st.dual_clip_fraction - want["dual_clip_fraction"]) * st.tokens <= 1


def test_actor_only_with_precomputed_old_ref(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(9)
    B, T, V = 6, 10, 32000
    lengths, tokens, mask, adv, rows = _random_case(rng, B, T, V, O.F32, masked=False)
    old = rng.uniform(-12, -1, (B, T)).astype(np.float32)
    ref = old + rng.uniform(-0.2, 0.2, (B, T)).astype(np.float32)
    cfg = rlo.TrainConfig(kl_coef=0.1)
    obj.ppo_gradient(cfg, dev(torch, tokens), dev(torch, lengths), dev(torch, rows[0]), dev(torch, adv),
                     old_logprobs=dev(torch, old), ref_logprobs=dev(torch, ref))
    st = obj.merge_gradients(cfg)
    lp, ent, _ = O.forward_logprobs(rows[0], O.F32, V, V, B, T, lengths, tokens)
    oc = O.TrainConfig(kl_coef=0.1)
    _, _, part = O.ppo_loss(oc, B, T, lengths, None, lp, old, ref, adv, ent)
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl"):
        assert close(getattr(st, k), want[k]), k


def test_micro_batches_and_determinism(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(4)
    B, T, V = 12, 9, 4096
    lengths, tokens, mask, adv, rows = _random_case(rng, B, T, V, O.F32)
    cfg = rlo.TrainConfig(kl_coef=0.02, loss_agg="group-mean", group_size=3)
    args = [dev(torch, x) for x in (tokens, lengths, rows[0], adv, mask, rows[1], rows[2])]

    def full():
        obj.ppo_gradient(cfg, args[0], args[1], args[2], args[3], mask=args[4], old_logits=args[5],
                         ref_logits=args[6])
        return obj.merge_gradients(cfg, with_partials=True)

    st1, p1 = full()
    st2, p2 = full()
    assert np.array_equal(p1, p2)  # bitwise reproducible (no float atomics)
    for s0, n in [(0, 6), (6, 3), (9, 3)]:  # whole-group micro-batches
        rs = slice(s0 * T, (s0 + n) * T)
        obj.ppo_gradient(cfg, args[0][s0:s0 + n], args[1][s0:s0 + n], args[2][rs], args[3][s0:s0 + n],
                         mask=args[4][s0:s0 + n], old_logits=args[5][rs], ref_logits=args[6][rs], seq_offset=s0)
    st3, p3 = obj.merge_gradients(cfg, with_partials=True)
    assert np.array_equal(p1, p3)
    assert st3.loss == st1.loss


def test_loss_error_paths_match_reference(env):
    torch, rlo, obj = env
    errs = golden("ppo_stats.json")["errors"]
    logits = dev(torch, np.zeros((1, 16), np.float32))
    one = dev(torch, np.array([1], np.int32))
    tok = dev(torch, np.array([[2]], np.int32))
    cfg = rlo.TrainConfig()
    lp = float(-math.log(16))
    obj.ppo_gradient(cfg, tok, one, logits, dev(torch, np.array([[0.5]], np.float32)),
                     mask=dev(torch, np.array([[0]], np.uint8)), old_logprobs=dev(torch, np.array([[lp]], np.float32)))
    with pytest.raises(rlo.TrainingError) as e:
        obj.merge_gradients(cfg)
    assert str(e.value) == errs["no_tokens"][1]
    obj.ppo_gradient(cfg, tok, one, logits, dev(torch, np.array([[np.nan]], np.float32)),
                     old_logprobs=dev(torch, np.array([[lp]], np.float32)))
    with pytest.raises(rlo.TrainingError) as e:
        obj.merge_gradients(cfg)
    assert str(e.value) == errs["nan_adv"][1]
    with pytest.raises(rlo.InputError, match="missing ref logprobs"):
        obj.ppo_gradient(rlo.TrainConfig(kl_coef=0.1), tok, one, logits, dev(torch, np.array([[0.5]], np.float32)),
                         old_logprobs=dev(torch, np.array([[lp]], np.float32)))
    # clipped-branch KAT, test_policy.cpp:357-379: loss = -(1+eps)*A, zero gradient
    adv = dev(torch, np.array([[2.0]], np.float32))
    outs = obj.ppo_gradient(cfg, tok, one, logits, adv, old_logprobs=dev(torch, np.array([[lp - 1.0]], np.float32)))
    st = obj.merge_gradients(cfg)
    assert close(st.loss, -2.4, 1e-6) and outs["dlogp"].item() == 0.0 and st.clip_fraction == 1.0


def test_step_host_matches_device_path(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(12)
    B, T, V = 8, 16, 8192
    lengths, tokens, mask, adv, rows = _random_case(rng, B, T, V, O.F32)
    rs = rng.integers(0, 2, B).astype(np.float32)
    cfg = rlo.TrainConfig(adv_estimator="grpo", group_size=4, kl_coef=0.01, kl_estimator="k3",
                          whiten_advantages=True)
    L = [dev(torch, r) for r in rows]
    st_dev = obj.step(cfg, dev(torch, tokens), dev(torch, lengths), L[0], mask=dev(torch, mask),
                      scalar_rewards=dev(torch, rs), old_logits=L[1], ref_logits=L[2])
    adv_h = np.zeros((B, T), np.float32)
    lp_h = np.zeros((B, T), np.float32)
    st_host = obj.step_host(cfg, tokens, lengths, L[0], mask=mask, scalar_rewards=rs, old_logits=L[1],
                            ref_logits=L[2], adv_out=adv_h, logp_out=lp_h)
    assert st_dev == st_host
    oc = O.TrainConfig(adv_estimator=O.GRPO, group_size=4, kl_coef=0.01, kl_estimator=O.K3, whiten_advantages=1)
    o_adv, _ = O.compute_advantages(oc, B, T, lengths, mask, None, rs.astype(np.float64))
    assert_close(adv_h.ravel(), o_adv, tol=2e-5, what="host adv")
    lps = [O.forward_logprobs(r, O.F32, V, V, B, T, lengths, tokens) for r in rows]
    m = (mask.ravel() != 0) & (np.arange(T)[None, :] < lengths[:, None]).ravel()
    assert_close(lp_h.ravel()[m], lps[0][0][m], what="host logp")
    _, _, part = O.ppo_loss(oc, B, T, lengths, mask, lps[0][0], lps[1][0], lps[2][0], o_adv, lps[0][1])
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "mean_kl"):
        assert close(getattr(st_host, k), want[k], 2e-5), k


def test_policy_worker_plugin(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(3)
    B, T, V = 4, 6, 1000
    lengths, tokens, mask, adv, rows = _random_case(rng, B, T, V, O.F32, masked=False)
    w = rlo.PolicyWorker(0, rlo.TrainConfig())
    batch = {"logits": dev(torch, rows[1]), "response_tokens": dev(torch, tokens), "lengths": dev(torch, lengths)}
    out = w.call("forward_logprobs", rlo.Message(batch=batch))
    old = out.batch["ref_logprobs"]  # the reference worker's scores
    lp, _, _ = O.forward_logprobs(rows[1], O.F32, V, V, B, T, lengths, tokens)
    assert_close(old.cpu().numpy().ravel(), lp)
    batch2 = {"logits": dev(torch, rows[0]), "response_tokens": batch["response_tokens"], "lengths": batch["lengths"],
              "response_logprobs": old, "advantages": dev(torch, adv)}
    rep = w.call("compute_gradient", rlo.Message(batch=batch2))
    assert rep.scalars["tokens"] == int(lengths.sum())
    assert len(rep.tensors["grad"]) == 0 and rep.tensors["dlogp"].shape == (B, T)
    with pytest.raises(rlo.DispatchError):
        w.call("generate", rlo.Message())
    # the reference controller's step over two workers (policy_workers.cpp:208-232):
    # rank-ordered merge of the shards == one worker over the whole batch, then
    # apply_update advances every worker's version (policy.cpp:452-460)
    seen = []
    ws = [rlo.PolicyWorker(0, rlo.TrainConfig(), rank=r, world_size=2,
                           on_update=lambda lr, g, v: seen.append((lr, len(g), v))) for r in range(2)]
    half = lambda d, s: {k: v[s] for k, v in d.items() if k != "logits"} | {  # noqa: E731
        "logits": d["logits"].view(B, T, V)[s].reshape(-1, V)}
    st2 = rlo.cluster_train_step(ws, [half(batch2, slice(0, 2)), half(batch2, slice(2, 4))], rlo.TrainConfig())
    st1 = rlo.merge_partials(np.array([[rep.scalars.get(k, 0.0) for k in ("loss_sum", "ratio_sum", "kl_sum")] +
                                       [0.0, rep.scalars["clipped"], 0.0, rep.scalars["tokens"]] + [0.0] * 9]),
                             rlo.TrainConfig())
    assert close(st2.loss, st1.loss, 1e-12) and st2.tokens == st1.tokens
    assert seen == [(0.05, 0, 2), (0.05, 0, 2)]
    assert all(w.call("get_version", rlo.Message()).fields["version"] == "2" for w in ws)


def test_full_size_config2_properties(env):
    """BASELINE config 2 shape (256 x 1024 tokens, V=32000 fp32, 3 logits
    tensors = 100 GB): size-independent properties + sampled oracle parity."""
    torch, rlo, obj = env
    B, T, V, seed = 256, 1024, 32000, 2
    free = torch.cuda.mem_get_info()[0]
    if free < 110e9:
        pytest.skip("needs ~105 GB of free HBM")
    L = [torch.empty(B * T, V, dtype=torch.float32, device="cuda") for _ in range(3)]
    for m in range(3):
        rlo.synth_logits(L[m], seed=seed, model=m)
    toks = torch.empty(B, T, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(toks, V, seed=seed)
    lengths = torch.full((B,), T, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(0)
    rw = dev(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32) * (rng.random((B, T)) < 0.01))
    vals = dev(torch, rng.standard_normal((B, T)).astype(np.float32) * 0.5)
    cfg = rlo.TrainConfig(adv_estimator="gae", lambd=0.95, kl_coef=0.001, kl_estimator="k3", whiten_advantages=True)
    adv = obj.compute_advantages(cfg, lengths, rewards=rw, values=vals)
    outs = obj.ppo_gradient(cfg, toks, lengths, L[0], adv, old_logits=L[1], ref_logits=L[2],
                            outputs=("logp", "old_logp", "ref_logp", "entropy", "loss"))
    st = obj.merge_gradients(cfg)
    # sampled rows against the oracle (rows regenerated on the CPU)
    idx = rng.choice(B * T, 48, replace=False)
    tk = toks.cpu().numpy().ravel()
    for name, m in (("logp", 0), ("old_logp", 1), ("ref_logp", 2)):
        got = outs[name].cpu().numpy().ravel()
        for r in idx[:16]:
            z = O.synth_row(O.F32, V, seed, m, int(r))
            lse, ent = O.logsoftmax_row(z)
            assert close(got[r], z[tk[r]] - lse), (name, r)
            if m == 0:
                assert close(outs["entropy"].cpu().numpy().ravel()[r], ent)
    # the full-size reduction against the oracle applied to the GPU's own per-token log-probs
    lp, old, ref, ent = (outs[k].cpu().numpy().ravel().astype(np.float64)
                         for k in ("logp", "old_logp", "ref_logp", "entropy"))
    oc = O.TrainConfig(adv_estimator=O.GAE, lambd=0.95, kl_coef=0.001, kl_estimator=O.K3, whiten_advantages=1)
    o_adv, _ = O.compute_advantages(oc, B, T, np.full(B, T, np.int32), None, rw.cpu().numpy().ravel().astype(np.float64),
                                    None, vals.cpu().numpy().ravel().astype(np.float64))
    assert_close(adv.cpu().numpy().ravel(), o_adv, tol=2e-5, what="full-size adv")
    _, _, part = O.ppo_loss(oc, B, T, np.full(B, T, np.int32), None, lp, old, ref,
                            adv.cpu().numpy().ravel().astype(np.float64), ent)
    want = O.merge(part[None], oc)
    for k in ("loss", "mean_ratio", "mean_kl", "mean_entropy"):
        assert close(getattr(st, k), want[k]), k
    assert st.tokens == B * T
    # ratio-one identity at full size (test_policy.cpp:339-355): old == actor, kl 0 -> loss = -mean(A)
    cfg1 = rlo.TrainConfig()
    obj.ppo_gradient(cfg1, toks, lengths, L[0], adv, old_logits=L[0])
    st1 = obj.merge_gradients(cfg1)
    # exactly 1 when both rows use the same exp2 path; within 1e-7 when the bf16 mix sends part of
    # the old-policy row's exponentials through the FMA-pipe polynomial (relative error <= 2.9e-6 per
    # term, on a quarter of the pairs)
    assert abs(st1.mean_ratio - 1.0) <= 1e-7 and close(st1.loss, -float(adv.double().mean()), 1e-6)
    del L
    torch.cuda.empty_cache()


def test_extensions_pinned_to_reference_identities(env):
    """GAE (lambda = 1) = the reference's discounted return minus the value;
    GRPO on one group of one-token samples = the reference's whitening; the
    entropy = -sum p log p of the reference's full log-softmax
    (tests/golden/extensions.json, made by the reference's own code)."""
    torch, rlo, obj = env
    ext = golden("extensions.json")
    for c in ext["gae_lambda1"]:
        B, T = c["B"], c["T"]
        cfg = rlo.TrainConfig(**{k: v for k, v in c["cfg"].items()})
        adv = obj.compute_advantages(cfg, dev(torch, np.asarray(c["lengths"], np.int32)), T=T,
                                     mask=dev(torch, np.asarray(c["mask"], np.uint8).reshape(B, T)),
                                     rewards=dev(torch, np.asarray(c["rewards_tok"], np.float32).reshape(B, T)),
                                     values=dev(torch, np.asarray(c["values"], np.float32).reshape(B, T)))
        assert_close(adv.cpu().numpy().ravel(), c["expect"], tol=2e-5, what="gae lambda=1")
    for c in ext["grpo_one_group"]:
        cfg = rlo.TrainConfig(**c["cfg"])
        adv = obj.compute_advantages(cfg, dev(torch, np.asarray(c["lengths"], np.int32)), T=c["T"],
                                     scalar_rewards=dev(torch, np.asarray(c["rewards_seq"], np.float32)))
        # fp32 rewards on the device: compare with the identity on the same fp32-rounded inputs
        rs = np.asarray(c["rewards_seq"], np.float32).astype(np.float64)
        want = np.clip((rs - rs.mean()) / (rs.std() + 1e-8), -10.0, 10.0)
        assert_close(adv.cpu().numpy().ravel(), want, tol=2e-5, what="grpo one group")
        assert_close(want, c["expect"], tol=1e-5, what="identity vs reference")
    for c in ext["entropy"]:
        row = np.asarray(c["row"], np.float32)
        out = obj.forward_logprobs(dev(torch, row[None, :]), dev(torch, np.zeros((1, 1), np.int32)),
                                   dev(torch, np.array([1], np.int32)), entropy=True)
        h = float(out["entropy"].item())
        assert abs(h - c["entropy"]) <= 1e-5 * max(1.0, abs(c["entropy"])), (c["V"], h, c["entropy"])


def test_aggregation_and_dual_clip_identities_on_gpu(env):
    """GPU seq-mean-token-mean / group-mean / never-binding dual-clip on
    equal-length unmasked batches reproduce the reference's token-mean loss."""
    torch, rlo, obj = env
    for c in golden("extensions.json")["aggregation"]:
        B, T = c["B"], c["T"]
        row = np.asarray(c["row"], np.float32)
        logits = dev(torch, np.tile(row, (B * T, 1)))
        for extra in (dict(loss_agg=1), dict(loss_agg=3, group_size=c["G"]), dict(dual_clip_c=1e9)):
            cfg = rlo.TrainConfig(**c["cfg"], **extra)
            obj.ppo_gradient(cfg, dev(torch, _arr(c["tokens"], np.int32).reshape(B, T)),
                             dev(torch, _arr(c["lengths"], np.int32)), logits, dev(torch, _arr(c["adv"]).reshape(B, T)),
                             old_logprobs=dev(torch, _arr(c["old"]).reshape(B, T)),
                             ref_logprobs=dev(torch, _arr(c["ref"]).reshape(B, T)))
            st = obj.merge_gradients(cfg)
            assert close(st.loss, c["ref_stats"]["loss"], tol=2e-5), (extra, st.loss, c["ref_stats"]["loss"])


def test_whole_step_in_a_cuda_graph(env):
    """compute_advantages -> ppo_gradient -> merge_gradients_async captured in
    a CUDA graph and replayed: the same UpdateStats as the synchronous step,
    fresh inputs picked up on replay, errors reported through the result."""
    torch, rlo, obj = env
    B, T, V, G = 8, 32, 4096, 4
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = [torch.randn(B * T, V, device="cuda", generator=gen) * 2 for _ in range(3)]
    K = torch.randint(0, V, (B, T), device="cuda", dtype=torch.int32, generator=gen)
    L = torch.tensor([T, T - 3, T, 5, T, 1, T, 9], dtype=torch.int32, device="cuda")
    M = torch.ones(B, T, dtype=torch.uint8, device="cuda")
    R = torch.rand(B, device="cuda", generator=gen)
    adv = torch.empty(B, T, device="cuda")
    res = torch.zeros(88, dtype=torch.uint8, device="cuda")
    cfg = rlo.TrainConfig(adv_estimator="grpo", group_size=G, kl_coef=0.01, kl_estimator="k3")

    def sync_step():
        obj.compute_advantages(cfg, L, T=T, mask=M, scalar_rewards=R, out=adv)
        obj.ppo_gradient(cfg, K, L, x[0], adv, mask=M, old_logits=x[1], ref_logits=x[2], outputs=())
        return obj.merge_gradients(cfg)

    def async_step():
        obj.compute_advantages(cfg, L, T=T, mask=M, scalar_rewards=R, out=adv)
        obj.ppo_gradient(cfg, K, L, x[0], adv, mask=M, old_logits=x[1], ref_logits=x[2], outputs=())
        obj.merge_gradients_async(cfg, out=res)

    want = sync_step()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        async_step()  # warm-up: every workspace buffer is sized before capture
    torch.cuda.synchronize()
    assert rlo.Objective.step_result(res) == want
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        async_step()
    res.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert rlo.Objective.step_result(res) == want
    R.copy_(torch.rand(B, device="cuda", generator=gen))  # new rewards, same buffers
    g.replay()
    torch.cuda.synchronize()
    got = rlo.Objective.step_result(res)
    assert got == sync_step() and got != want
    M.zero_()  # no participating token: the reference's TrainingError, through the result
    g.replay()
    torch.cuda.synchronize()
    with pytest.raises(rlo.TrainingError, match="no loss-participating tokens"):
        rlo.Objective.step_result(res)
