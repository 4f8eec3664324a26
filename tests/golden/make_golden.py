"""Generate the golden fixtures under tests/golden/ from the REFERENCE'S OWN
code (oracle/_ref/librollmini_ref.so, built by oracle/Makefile from
/root/reference/proj/core/src).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The GPU box never needs /root/reference: tests read only the committed
fixtures.  Every fixture records which reference function produced it.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def logsoftmax_cases(rng):
    """policy.cpp:116-122 via next_token_forward (b2 trick)."""
    rows32, toks32, lp32, Vs = [], [], [], []
    for V, scale in [(9, 0.0), (9, 1.0), (57, 3.0), (1000, 3.0), (1000, 40.0), (4099, 8.0)]:
        for _ in range(3):
            z = (rng.standard_normal(V) * scale).astype(np.float32)
            if V >= 57:
                z[rng.integers(0, V, 3)] += np.float32(12.0)
            tok = int(rng.integers(0, V))
            lp = O.ref_logsoftmax_rows(z.astype(np.float64), [tok])[0]
            rows32.append(z)
            toks32.append(tok)
            lp32.append(lp)
            Vs.append(V)
    # synthetic rows (include/rlo_synth.h), regenerated from keys at test time
    synth = []
    for dtype, V, seed, model, key in [(O.F32, 32000, 7, 0, 3), (O.F32, 32000, 7, 1, 3), (O.F32, 32000, 7, 2, 3),
                                       (O.BF16, 152064, 11, 0, 5), (O.BF16, 152064, 11, 2, 6),
                                       (O.BF16, 4096, 5, 1, 0)]:
        row = O.synth_row(dtype, V, seed, model, key)
        tok = O.synth_token(seed, key, V)
        lp = O.ref_logsoftmax_rows(row, [tok])[0]
        synth.append(dict(dtype=dtype, V=V, seed=seed, model=model, key=key, token=tok, ref_lp=lp,
                          row_sum=float(row.sum()), row_max=float(row.max())))
    flat = np.concatenate(rows32)
    offs = np.cumsum([0] + Vs[:-1])
    np.savez_compressed(os.path.join(HERE, "logsoftmax.npz"), rows=flat, offsets=np.array(offs), V=np.array(Vs),
                        tokens=np.array(toks32, dtype=np.int32), ref_lp=np.array(lp32))
    with open(os.path.join(HERE, "logsoftmax_synth.json"), "w") as f:
        json.dump({"source": "policy.cpp:116-122 via next_token_forward, PolicyLayout{V,1,1,1}, b2=row",
                   "cases": synth}, f, indent=1)


def forward_logprobs_case(rng):
    """forward_logprobs itself (policy.cpp:210-233), one shared row."""
    V, B, T = 33, 5, 7
    row = rng.standard_normal(V).astype(np.float32)
    lengths = np.array([7, 0, 3, 5, 1], dtype=np.int32)
    tokens = rng.integers(0, V, B * T).astype(np.int32)
    lp = O.ref_forward_logprobs_b2(row.astype(np.float64), B, T, lengths, tokens)
    bad = tokens.copy()
    bad[2 * T + 1] = V  # out of vocabulary in a valid position
    try:
        O.ref_forward_logprobs_b2(row.astype(np.float64), B, T, lengths, bad)
        msg = None
    except O.OracleError as e:
        msg = (e.code, str(e))
    np.savez_compressed(os.path.join(HERE, "forward_logprobs.npz"), row=row, lengths=lengths, tokens=tokens,
                        ref_lp=lp, bad_tokens=bad)
    return {"oov_error": msg}


def advantage_cases(rng):
    """compute_advantages (policy.cpp:257-311)."""
    cases = []

    def add(name, cfg_kw, B, T, lengths, mask=None, rewards_tok=None, rewards_seq=None):
        cfg = O.TrainConfig(**cfg_kw)
        try:
            out = O.ref_compute_advantages(cfg, B, T, lengths, mask, rewards_tok, rewards_seq)
            err = None
        except O.OracleError as e:
            out, err = None, [e.code, str(e)]
        cases.append(dict(name=name, cfg=cfg_kw, B=B, T=T, lengths=np.asarray(lengths).tolist(),
                          mask=None if mask is None else np.asarray(mask).tolist(),
                          rewards_tok=None if rewards_tok is None else np.asarray(rewards_tok).tolist(),
                          rewards_seq=None if rewards_seq is None else np.asarray(rewards_seq).tolist(),
                          ref_adv=None if out is None else out.tolist(), error=err))

    # test_policy.cpp:229-236 terminal reward, gamma 1 -> [1,1,1]
    add("kat_terminal", dict(gamma=1.0), 1, 3, [3], rewards_seq=[1.0])
    # test_policy.cpp:240-249 [0,0,30] -> clip 20 -> adv clip 10
    add("kat_clip", dict(gamma=1.0, reward_clip=20.0, advantage_clip=10.0), 1, 3, [3], rewards_tok=[0.0, 0.0, 30.0])
    # test_policy.cpp:252-257 missing rewards -> InputError
    add("kat_missing", dict(), 1, 1, [1])
    # test_policy.cpp:281-304 whitening over 4 seqs with terminal rewards 0..3
    add("kat_whiten", dict(whiten_advantages=1, advantage_clip=100.0), 4, 4, [4, 4, 4, 4],
        rewards_tok=np.concatenate([[0, 0, 0, float(i)] for i in range(4)]))
    for k in range(6):
        B, T = int(rng.integers(3, 9)), int(rng.integers(4, 24))
        lengths = rng.integers(0, T + 1, B)
        lengths[0] = T
        mask = (rng.random(B * T) < 0.7).astype(np.uint8)
        kw = dict(gamma=float(rng.choice([1.0, 0.9, 0.97])), whiten_advantages=int(k % 2),
                  reward_clip=float(rng.choice([20.0, 0.5])), advantage_clip=float(rng.choice([10.0, 0.8])))
        if k < 3:
            rt = rng.standard_normal(B * T) * 2.0
            rt[rng.integers(0, B * T)] = 35.0
            add(f"random_tok_{k}", kw, B, T, lengths, mask, rewards_tok=rt)
        else:
            add(f"random_seq_{k}", kw, B, T, lengths, mask if k != 4 else None,
                rewards_seq=rng.standard_normal(B) * 3.0)
    with open(os.path.join(HERE, "advantages.json"), "w") as f:
        json.dump({"source": "compute_advantages policy.cpp:257-311", "cases": cases}, f)


def ppo_cases(rng):
    """ppo_gradient -> merge_gradients stats (policy.cpp:313-450), b2 trick."""
    cases = []
    for k in range(8):
        V = int(rng.choice([9, 17, 64]))
        B, T = int(rng.integers(2, 8)), int(rng.integers(2, 10))
        row = rng.standard_normal(V) * 1.5
        lengths = rng.integers(1, T + 1, B)
        tokens = rng.integers(0, V, B * T).astype(np.int32)
        mask = (rng.random(B * T) < 0.8).astype(np.uint8) if k % 2 else None
        full = O.ref_logsoftmax_rows(row, [0], full=True)[1][0]
        lp = full[tokens]
        old = lp + rng.uniform(-0.4, 0.4, B * T)
        ref_lp = lp + rng.uniform(-0.3, 0.3, B * T)
        adv = rng.uniform(-1, 1, B * T)
        adv += np.where(adv >= 0, 0.3, -0.3)
        kw = dict(clip_eps=float(rng.choice([0.1, 0.2, 0.3])), kl_coef=float(rng.choice([0.0, 0.1])))
        world = int(rng.choice([1, 2, 3]))
        st = O.ref_ppo_stats_b2(row, B, T, lengths, tokens, mask, old, ref_lp, adv, O.TrainConfig(**kw), world)
        # merged gradient w.r.t. the shared logits row (policy.cpp:375-379, :391, :439-440)
        grad = O.ref_ppo_grad_b2(row, B, T, lengths, tokens, mask, old, ref_lp, adv, O.TrainConfig(**kw), world)
        cases.append(dict(cfg=kw, V=V, B=B, T=T, world=world, row=row.tolist(), lengths=lengths.tolist(),
                          tokens=tokens.tolist(), mask=None if mask is None else mask.tolist(), old=old.tolist(),
                          ref=ref_lp.tolist(), adv=adv.tolist(), ref_stats=st, ref_grad_row=grad.tolist()))
    # clipped-branch KAT (test_policy.cpp:357-379): ratio=e^1 >> 1.2, A=2 -> loss -2.4
    V = 9
    row = rng.standard_normal(V)
    full = O.ref_logsoftmax_rows(row, [0], full=True)[1][0]
    st = O.ref_ppo_stats_b2(row, 1, 1, [1], [2], None, [full[2] - 1.0], None, [2.0], O.TrainConfig(), 1)
    cases.append(dict(cfg={}, V=V, B=1, T=1, world=1, row=row.tolist(), lengths=[1], tokens=[2], mask=None,
                      old=[full[2] - 1.0], ref=None, adv=[2.0], ref_stats=st, kat="clipped_branch"))
    # error paths (policy.cpp:437, 441)
    errors = {}
    for name, adv0, mask in [("no_tokens", 0.5, [0]), ("nan_adv", float("nan"), None)]:
        try:
            O.ref_ppo_stats_b2(row, 1, 1, [1], [2], mask, [full[2]], None, [adv0], O.TrainConfig(), 1)
            errors[name] = None
        except O.OracleError as e:
            errors[name] = [e.code, str(e)]
    with open(os.path.join(HERE, "ppo_stats.json"), "w") as f:
        json.dump({"source": "ppo_gradient+merge_gradients policy.cpp:313-450 (b2 trick)", "cases": cases,
                   "errors": errors}, f)


def value_cases(rng):
    """value_gradient (policy.cpp:474-540): every position's value = vb (value-head bias)."""
    cases = []
    for k in range(5):
        B, T = int(rng.integers(2, 7)), int(rng.integers(2, 12))
        lengths = rng.integers(0, T + 1, B).astype(np.int32)
        lengths[0] = T
        mask = (rng.random(B * T) < 0.75).astype(np.uint8) if k % 2 else None
        targets = rng.standard_normal(B * T) * 2.0
        vb = float(rng.standard_normal())
        r = O.ref_value_loss_b2(vb, B, T, lengths, mask, targets)
        cases.append(dict(B=B, T=T, vb=vb, lengths=lengths.tolist(), mask=None if mask is None else mask.tolist(),
                          targets=targets.tolist(), ref=r))
    with open(os.path.join(HERE, "value_loss.json"), "w") as f:
        json.dump({"source": "value_gradient policy.cpp:474-540 (value = vb everywhere)", "cases": cases}, f)


def decode_cases(rng):
    """decode_next (policy.cpp:143-169) through the reference's own code (b2 trick)."""
    cases = []
    rows = []
    for k in range(12):
        V = int(rng.choice([9, 52, 1000, 2053]))
        scale = float(rng.choice([0.5, 2.0, 4.0]))
        row = (rng.standard_normal(V) * scale).astype(np.float32).astype(np.float64)
        for _ in range(16):
            T = float(rng.choice([0.3, 0.7, 1.0, 1.5]))
            seed, version = int(rng.integers(0, 2**63)), int(rng.integers(1, 50))
            sid = f"s{int(rng.integers(0, 10**6))}"
            key, pos = O.ref_hash_str(sid), int(rng.integers(0, 4096))
            tok, lp = O.ref_decode_b2(row, T, seed, version, key, pos)
            cases.append(dict(row=len(rows), temperature=T, seed=seed, version=version, sample_id=sid, sample_key=key,
                              position=pos, ref_token=tok, ref_logp=lp))
        rows.append(row.tolist())
    with open(os.path.join(HERE, "decode.json"), "w") as f:
        json.dump({"source": "decode_next policy.cpp:143-169 (b2 trick), hash_str rng.hpp:34-41", "rows": rows,
                   "cases": cases}, f)


def jsonl_cases():
    """SampleBatch::to_jsonl (sample.cpp:144-148): the reference's own wire text."""
    with open(os.path.join(HERE, "batch.jsonl"), "w", encoding="utf-8") as f:
        f.write(O.ref_batch_jsonl(2506, 40))
    bad = {
        "duplicate_id": '{"sample_id":"a","response_tokens":[1]}\n{"sample_id":"a","response_tokens":[2]}\n',
        "length_mismatch": '{"sample_id":"x","response_tokens":[1,2,3],"rewards":[0.0,1.0]}\n',
        "mask_mismatch": '{"sample_id":"y","response_tokens":[1,2],"action_mask":[1]}\n',
    }
    jsonl_errors = {k: list(O.ref_parse_validate_jsonl(v)) + [v] for k, v in bad.items()}
    plans = [dict(total=t, bucket=b, plan=O.ref_bucket_plan(t, b))
             for t, b in [(1000, 256), (0, 7), (7, 7), (8, 7), (207, 1), (1 << 20, 65536), (1000003, 4096)]]
    return {"bucket_plan": plans, "jsonl_errors": jsonl_errors}


def config_cases():
    """TrainConfig::validate messages (policy.cpp:29-37) and split_sizes (sample.cpp:99-105)."""
    bad = [dict(clip_eps=0.0), dict(clip_eps=1.0), dict(kl_coef=-0.1), dict(learning_rate=-1.0),
           dict(advantage_clip=0.0), dict(reward_clip=-1.0), dict(gamma=0.0), dict(gamma=1.5), {}]
    out = []
    for kw in bad:
        code, msg = O.ref_train_config_validate(O.TrainConfig(**kw))
        out.append(dict(cfg=kw, code=code, msg=msg))
    splits = []
    for n, w in [(8, 4), (10, 4), (7, 1), (3, 5), (0, 3), (1001, 8)]:
        splits.append(dict(n=n, parts=w, sizes=O.ref_split_sizes(n, w).tolist()))
    return out, splits


def extension_cases(rng):
    """Pin the extensions the reference lacks to its own code where an identity
    exists: GAE with lambda = 1 telescopes to the reference's discounted
    return minus the value; GRPO on one group of one-token samples with
    eps = 1e-8 is the reference's whitening; the entropy of a row is
    -sum p log p over the reference's own full log-softmax."""
    gae, grpo, ent = [], [], []
    for k in range(4):
        B, T = int(rng.integers(2, 7)), int(rng.integers(3, 20))
        lengths = rng.integers(0, T + 1, B)
        lengths[0] = T
        mask = (rng.random(B * T) < 0.7).astype(np.uint8)
        g = float(rng.choice([1.0, 0.9, 0.99]))
        rt = rng.standard_normal(B * T) * 2.0
        vals = rng.standard_normal(B * T) * 0.5
        kw = dict(gamma=g, reward_clip=1e6, advantage_clip=1e9)
        ref = O.ref_compute_advantages(O.TrainConfig(**kw), B, T, lengths, mask, rewards_tok=rt)
        valid = (np.arange(T)[None, :] < lengths[:, None]).ravel()
        expect = np.where(valid, ref - vals, 0.0)
        gae.append(dict(cfg=dict(kw, adv_estimator=2, lambd=1.0), B=B, T=T, lengths=lengths.tolist(),
                        mask=mask.tolist(), rewards_tok=rt.tolist(), values=vals.tolist(), expect=expect.tolist()))
    for B in (4, 8, 16):
        rs = rng.standard_normal(B) * 2.0
        kw = dict(advantage_clip=10.0, reward_clip=20.0)
        ref = O.ref_compute_advantages(O.TrainConfig(whiten_advantages=1, **kw), B, 1, [1] * B, None, rewards_seq=rs)
        grpo.append(dict(cfg=dict(kw, adv_estimator=1, group_size=B, grpo_eps=1e-8), B=B, T=1, lengths=[1] * B,
                         rewards_seq=rs.tolist(), expect=ref.tolist()))
    for V, scale in [(9, 1.0), (57, 3.0), (1000, 3.0), (4099, 8.0), (8192, 3.0)]:
        z = (rng.standard_normal(V) * scale).astype(np.float32)
        _, full = O.ref_logsoftmax_rows(z.astype(np.float64), [0], full=True)
        lp = full[0]
        ent.append(dict(V=V, row=z.tolist(), entropy=float(-(np.exp(lp) * lp).sum())))
    # aggregation / dual-clip identities: with equal lengths and no mask every
    # sequence and group holds the same token count, so seq-mean-token-mean and
    # group-mean equal the reference's token-mean; a dual-clip cap that never
    # binds (c = 1e9) leaves the reference's clipped surrogate unchanged
    agg = []
    for k in range(4):
        V, G = int(rng.choice([17, 64])), int(rng.choice([2, 3]))
        B, T = G * int(rng.integers(1, 4)), int(rng.integers(2, 9))
        row = rng.standard_normal(V) * 1.5
        lengths = np.full(B, T)
        tokens = rng.integers(0, V, B * T).astype(np.int32)
        full = O.ref_logsoftmax_rows(row, [0], full=True)[1][0]
        lp = full[tokens]
        old = lp + rng.uniform(-0.4, 0.4, B * T)
        ref_lp = lp + rng.uniform(-0.3, 0.3, B * T)
        adv = rng.uniform(-1, 1, B * T)
        kw = dict(clip_eps=0.2, kl_coef=float(rng.choice([0.0, 0.1])))
        st = O.ref_ppo_stats_b2(row, B, T, lengths, tokens, None, old, ref_lp, adv, O.TrainConfig(**kw), 1)
        agg.append(dict(cfg=kw, G=G, V=V, B=B, T=T, row=row.tolist(), lengths=lengths.tolist(), tokens=tokens.tolist(),
                        old=old.tolist(), ref=ref_lp.tolist(), adv=adv.tolist(), ref_stats=st))
    with open(os.path.join(HERE, "extensions.json"), "w") as f:
        json.dump({"source": "identities onto compute_advantages policy.cpp:257-311 (GAE lambda=1, GRPO one group "
                             "of T=1 samples = whitening) and the full log-softmax policy.cpp:116-122 (entropy)",
                   "gae_lambda1": gae, "grpo_one_group": grpo, "entropy": ent, "aggregation": agg}, f)


def main():
    O.build(with_ref=True)
    rng = np.random.default_rng(20250606)
    logsoftmax_cases(rng)
    extra = forward_logprobs_case(rng)
    advantage_cases(rng)
    ppo_cases(rng)
    value_cases(np.random.default_rng(474))
    decode_cases(np.random.default_rng(143))
    extension_cases(np.random.default_rng(2506))
    extra.update(jsonl_cases())
    cfgs, splits = config_cases()
    with open(os.path.join(HERE, "misc.json"), "w") as f:
        json.dump({"train_config_validate": cfgs, "split_sizes": splits, **extra}, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
