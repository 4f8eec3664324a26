"""The N>1 data-parallel path on CPU: world_size-2 torch.distributed (gloo)
processes run the path's host logic exactly as the GPU ranks do —
group-aligned sharding (rlo_shard_plan), all-gather of the whitening
statistics and their rank-ordered combine (rlo_whiten_combine, the same code
the device normalise pass runs), all-gather of the per-rank partials and the
rank-ordered merge (rlo_merge_partials) — with the CPU oracle standing in
for each rank's device kernels.  The merged result must equal the
single-process oracle on the whole batch (DP equivalence, SPEC.md:267;
test_policy.cpp:478-497)."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(seed=7):
    rng = np.random.default_rng(seed)
    B, T, V, G = 24, 11, 64, 4
    lengths = rng.integers(1, T + 1, B).astype(np.int32)
    mask = (rng.random((B, T)) < 0.8).astype(np.uint8)
    rseq = rng.integers(0, 2, B).astype(np.float64)
    rows = rng.standard_normal((3, B * T, V)) * 2
    rows[1:] = rows[0] + rng.standard_normal((2, B * T, V)) * 0.1
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    return B, T, V, G, lengths, mask, rseq, rows.astype(np.float32), tokens


def _cfgs(O, agg):
    kw = dict(adv_estimator=O.GRPO, group_size=4, whiten_advantages=1, kl_coef=0.05, kl_estimator=O.K3,
              loss_agg=agg, dual_clip_c=3.0, advantage_clip=2.5)
    return kw


def _rank_main(rank, world, port, agg, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2506_06122_b200 as rlo
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, T, V, G, lengths, mask, rseq, rows, tokens = _problem()
        kw = _cfgs(O, agg)
        oc = O.TrainConfig(**kw)
        b0, n = rlo.shard_plan(B, G, world, rank)
        sl = slice(b0 * T, (b0 + n) * T)
        # rank-local raw advantages (whitening is global: done below)
        raw, _ = O.compute_advantages(O.TrainConfig(**{**kw, "whiten_advantages": 0, "advantage_clip": 1e30}),
                                      n, T, lengths[b0:b0 + n], mask[b0:b0 + n], None, rseq[b0:b0 + n])
        valid = (np.arange(T)[None, :] < lengths[b0:b0 + n, None]).ravel()
        m = valid & (mask[b0:b0 + n].ravel() != 0)
        local = torch.tensor([raw[m].sum(), (raw[m] ** 2).sum(), float(m.sum()), 0.0], dtype=torch.float64)
        gathered = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, local)
        apply, mean, inv = rlo.whiten_combine(torch.stack(gathered).numpy())
        adv = np.where(valid, (raw - mean) * inv if apply else raw, 0.0)
        adv = np.clip(adv, -kw["advantage_clip"], kw["advantage_clip"])
        lps = [O.forward_logprobs(r[sl], O.F32, V, V, n, T, lengths[b0:b0 + n], tokens[b0:b0 + n]) for r in rows]
        _, _, part = O.ppo_loss(oc, n, T, lengths[b0:b0 + n], mask[b0:b0 + n], lps[0][0], lps[1][0], lps[2][0], adv,
                                lps[0][1])
        parts = [torch.zeros(16, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor(part))
        st = rlo.merge_partials(torch.stack(parts).numpy(), rlo.TrainConfig(
            adv_estimator="grpo", group_size=4, whiten_advantages=True, kl_coef=0.05, kl_estimator="k3",
            loss_agg=agg, dual_clip_c=3.0, advantage_clip=2.5))
        out_q.put((rank, adv.tolist(), st.__dict__))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("agg", [0, 1, 3])
def test_two_rank_gloo_matches_single_process(agg):
    import torch.multiprocessing as mp

    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, agg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, adv, st = q.get(timeout=240)
        res[r] = (np.array(adv), st)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle on the whole batch
    B, T, V, G, lengths, mask, rseq, rows, tokens = _problem()
    oc = O.TrainConfig(**_cfgs(O, agg))
    adv, _ = O.compute_advantages(oc, B, T, lengths, mask, None, rseq)
    lps = [O.forward_logprobs(r, O.F32, V, V, B, T, lengths, tokens) for r in rows]
    _, _, part = O.ppo_loss(oc, B, T, lengths, mask, lps[0][0], lps[1][0], lps[2][0], adv, lps[0][1])
    want = O.merge(part[None], oc)
    np.testing.assert_allclose(np.concatenate([res[0][0], res[1][0]]), adv, rtol=1e-12, atol=1e-12)
    for r in range(world):
        st = res[r][1]
        for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl", "mean_entropy", "dual_clip_fraction"):
            assert st[k] == pytest.approx(want[k], rel=1e-12, abs=1e-14), k
        for k in ("tokens", "seqs", "groups"):
            assert st[k] == want[k]
