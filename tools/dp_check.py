"""Multi-GPU data-parallel parity check (run under torchrun, one process per GPU).

Every rank takes its group-aligned shard (rlo_shard_plan) of one
deterministic global batch, runs the whole path with an NCCL communicator
(global whitening statistics and loss partials all-gathered, merged in rank
order), and rank 0 compares against a single-GPU run of the full batch on its
own device (a second handle without a communicator): advantages within 1e-6,
stats within 1e-9 relative, counts exact — the reference's DP-equivalence
property (test_policy.cpp:478-497).  Prints PASS/FAIL lines and
exits non-zero on failure.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dp_check.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_06122_b200 as rlo  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    B, T, V, G = 48, 64, 8192, 4
    rng = np.random.default_rng(11)
    lengths = rng.integers(T // 4, T + 1, B).astype(np.int32)
    mask = (rng.random((B, T)) < 0.9).astype(np.uint8)
    rs = rng.integers(0, 2, B).astype(np.float32)
    cfgs = {
        "grpo+whiten+group-mean": rlo.TrainConfig(adv_estimator="grpo", group_size=G, whiten_advantages=True,
                                                  kl_coef=0.01, kl_estimator="k3", loss_agg="group-mean",
                                                  dual_clip_c=3.0),
        "gae+whiten+seq-mean": rlo.TrainConfig(adv_estimator="gae", group_size=G, whiten_advantages=True,
                                               gamma=0.99, lambd=0.95, kl_coef=0.05, kl_estimator="k2",
                                               loss_agg="seq-mean-token-mean"),
    }
    rt = (rng.standard_normal((B, T)) * 0.2).astype(np.float32)
    vals = (rng.standard_normal((B, T)) * 0.5).astype(np.float32)
    full = [torch.empty(B * T, V, dtype=torch.bfloat16, device=dev) for _ in range(3)]
    for m in range(3):
        rlo.synth_logits(full[m], seed=3, model=m)
    toks = torch.empty(B, T, dtype=torch.int32, device=dev)
    rlo.synth_tokens(toks, V, seed=3)

    obj = rlo.Objective(local)
    uid = [rlo.Objective.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    obj.init_comm(uid[0], rank, world)
    b0, n = rlo.shard_plan(B, G, world, rank)
    fails = 0
    for name, cfg in cfgs.items():
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        kw = dict(rewards=d(rt[b0:b0 + n]), values=d(vals[b0:b0 + n])) if cfg.adv_estimator == "gae" else \
            dict(scalar_rewards=d(rs[b0:b0 + n]))
        adv = obj.compute_advantages(cfg, d(lengths[b0:b0 + n]), T=T, mask=d(mask[b0:b0 + n]), **kw)
        rows = slice(b0 * T, (b0 + n) * T)
        obj.ppo_gradient(cfg, toks[b0:b0 + n].contiguous(), d(lengths[b0:b0 + n]), full[0][rows], adv,
                         mask=d(mask[b0:b0 + n]), old_logits=full[1][rows], ref_logits=full[2][rows])
        st = obj.merge_gradients(cfg)
        gathered = [torch.zeros(B, T, device=dev) for _ in range(world)] if rank == 0 else None
        pad = torch.zeros(B, T, device=dev)
        pad[:n] = adv
        dist.gather(pad, gathered, dst=0)
        counts = [None] * world
        dist.all_gather_object(counts, n)
        if rank == 0:
            single = rlo.Objective(local)
            kw1 = dict(rewards=d(rt), values=d(vals)) if cfg.adv_estimator == "gae" else dict(scalar_rewards=d(rs))
            adv1 = single.compute_advantages(cfg, d(lengths), T=T, mask=d(mask), **kw1)
            single.ppo_gradient(cfg, toks, d(lengths), full[0], adv1, mask=d(mask), old_logits=full[1],
                                ref_logits=full[2])
            st1 = single.merge_gradients(cfg)
            adv_dp = torch.cat([g[:c] for g, c in zip(gathered, counts)])
            a_err = float((adv_dp - adv1).abs().max())
            ok = a_err <= 1e-6
            for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl", "mean_entropy", "dual_clip_fraction"):
                g, r = getattr(st, k), getattr(st1, k)
                ok &= abs(g - r) <= 1e-9 * max(1.0, abs(r))
            ok &= (st.tokens, st.seqs, st.groups) == (st1.tokens, st1.seqs, st1.groups)
            print(f"{'PASS' if ok else 'FAIL'} dp{world} {name}: loss {st.loss:.12f} vs single {st1.loss:.12f}, "
                  f"adv max err {a_err:.2e}, tokens {st.tokens}", flush=True)
            fails += not ok
            single.close()
    # fused update pass: global counts (all-gathered) -> weights -> loss + dlogits
    # in one read of the actor logits; shards' gradient rows == the single run's
    cfg = cfgs["gae+whiten+seq-mean"]
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    Ls, Ms = d(lengths[b0:b0 + n]), d(mask[b0:b0 + n])
    adv = obj.compute_advantages(cfg, Ls, T=T, mask=Ms, rewards=d(rt[b0:b0 + n]), values=d(vals[b0:b0 + n]))
    cnt = obj.batch_counts(cfg, Ls, T, mask=Ms)
    w = obj.loss_weights(cfg, Ls, cnt, T, mask=Ms)
    rows = slice(b0 * T, (b0 + n) * T)
    _, g = obj.ppo_gradient_fused(cfg, toks[b0:b0 + n].contiguous(), Ls, full[0][rows], adv, w, mask=Ms,
                                  old_logits=full[1][rows], ref_logits=full[2][rows])
    st = obj.merge_gradients(cfg)
    gpad = torch.zeros(B * T, V, dtype=g.dtype, device=dev)
    gpad[: n * T] = g
    gathered = [torch.zeros_like(gpad) for _ in range(world)] if rank == 0 else None
    dist.gather(gpad, gathered, dst=0)
    counts = [None] * world
    dist.all_gather_object(counts, n)
    if rank == 0:
        single = rlo.Objective(local)
        adv1 = single.compute_advantages(cfg, d(lengths), T=T, mask=d(mask), rewards=d(rt), values=d(vals))
        cnt1 = single.batch_counts(cfg, d(lengths), T, mask=d(mask))
        w1 = single.loss_weights(cfg, d(lengths), cnt1, T, mask=d(mask))
        _, g1 = single.ppo_gradient_fused(cfg, toks, d(lengths), full[0], adv1, w1, mask=d(mask),
                                          old_logits=full[1], ref_logits=full[2])
        st1 = single.merge_gradients(cfg)
        g_dp = torch.cat([x[: c * T] for x, c in zip(gathered, counts)])
        g_err = float((g_dp.float() - g1.float()).abs().max())
        ok = (cnt.tokens, cnt.seqs, cnt.groups) == (cnt1.tokens, cnt1.seqs, cnt1.groups) and g_err <= 1e-6
        ok &= abs(st.loss - st1.loss) <= 1e-9 * max(1.0, abs(st1.loss))
        print(f"{'PASS' if ok else 'FAIL'} dp{world} fused update pass: counts {cnt.tokens}/{cnt.seqs}/{cnt.groups}, "
              f"dlogits max err {g_err:.2e}, loss {st.loss:.12f} vs {st1.loss:.12f}", flush=True)
        fails += not ok
        single.close()
    # device-side (graph-capturable) merge over NCCL == the synchronous merge
    cfg = cfgs["grpo+whiten+group-mean"]
    Ls, Ms = d(lengths[b0:b0 + n]), d(mask[b0:b0 + n])

    def body():
        adv = obj.compute_advantages(cfg, Ls, T=T, mask=Ms, scalar_rewards=d(rs[b0:b0 + n]))
        obj.ppo_gradient(cfg, toks[b0:b0 + n].contiguous(), Ls, full[0][rows], adv, mask=Ms,
                         old_logits=full[1][rows], ref_logits=full[2][rows], outputs=())
    body()
    st_sync = obj.merge_gradients(cfg)
    body()
    res = obj.merge_gradients_async(cfg)
    st_async = rlo.Objective.step_result(res)
    ok = st_sync == st_async
    okt = torch.tensor([int(ok)], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        good = bool(okt.item())
        print(f"{'PASS' if good else 'FAIL'} dp{world} async (device-side) merge == synchronous merge: "
              f"loss {st_async.loss:.12f}", flush=True)
        fails += not good
    # ModelUpdateGroup: bucketed broadcast, destinations bit-identical for every
    # bucket size (test_policy_workers.cpp:100-130's sync_params property)
    n_params = 1_000_003
    for bucket in (4, 28, 4096, 1 << 20, 4 * n_params):
        gen = torch.Generator(device=dev).manual_seed(1234)
        src = torch.randn(n_params, device=dev, generator=gen)
        buf = src.clone() if rank == 0 else torch.zeros_like(src)
        obj.broadcast_params(buf, bucket_bytes=bucket, root=0)
        ok = bool(torch.equal(buf, src))  # every rank can regenerate rank 0's values
        okt = torch.tensor([int(ok)], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if rank == 0:
            good = bool(okt.item())
            print(f"{'PASS' if good else 'FAIL'} dp{world} broadcast_params bucket={bucket} bytes: bit-identical", flush=True)
            fails += not good
    obj.close()
    flag = torch.tensor([fails], device=dev)
    dist.broadcast(flag, src=0)
    dist.destroy_process_group()
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
