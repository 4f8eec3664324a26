"""Every kernel librlo.so ships, on small shapes, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_cases.py

Launches (through the Python ctypes mirror of the C ABI): every vocab-pass
instantiation (fp32 / bf16 forward_logprobs with and without entropy; the
loss pass at P = 1, 2, 3 for both dtypes; the bf16 long-row lazy-max kernel
and the short-row lockstep kernel; -inf rows for the guarded entropy redo;
unaligned rows), the fused update pass (fp32 cluster kernel with DSMEM and
named barriers at NB = 2, and the forced bf16 8-CTA cluster), the backward
epilogue (fp32 / fp64 lse), the advantage scans (REINFORCE, GAE, GRPO, with
whitening), the per-sequence / batch reductions and the device-side merge
(merge_gradients_async), value loss, batch counts / loss weights, decode
(screen + fp64 redo), the synthetic generators.  Prints "sanitize cases ok".
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_06122_b200 as rlo  # noqa: E402


def main():
    obj = rlo.Objective(0)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731

    def logits(rows, V, dt, stride=None, seed=0, model=0):
        x = torch.empty(rows, stride or V, dtype=dt, device=dev)
        rlo.synth_logits(x, seed=seed, model=model)
        return x[:, :V]

    B, T = 4, 3
    lengths = t(np.array([3, 1, 0, 2], np.int32))
    m = (rng.random((B, T)) < 0.8).astype(np.uint8)
    m[0, :2] = 1  # at least two loss-participating tokens
    mask = t(m)
    for dt, V, stride in [(torch.float32, 4096, None), (torch.float32, 1001, 1001), (torch.bfloat16, 152064, None),
                          (torch.bfloat16, 4096, None), (torch.bfloat16, 50257, 50257)]:
        toks = t(rng.integers(0, V, (B, T)).astype(np.int32))
        L = [logits(B * T, V, dt, stride, model=m) for m in range(3)]
        L[0][1, ::7] = float("-inf")  # guarded entropy redo
        for ent in (False, True):
            obj.forward_logprobs(L[0], toks, lengths, entropy=ent)
        adv = t(rng.uniform(-1, 1, (B, T)).astype(np.float32))
        old = t(rng.uniform(-9, -1, (B, T)).astype(np.float32))
        cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3", dual_clip_c=3.0)
        for P in (1, 2, 3):
            kw = dict(old_logits=L[1]) if P >= 2 else dict(old_logprobs=old)
            if P >= 3:
                kw["ref_logits"] = L[2]
            else:
                kw["ref_logprobs"] = old
            obj.ppo_gradient(cfg, toks, lengths, L[0], adv, mask=mask,
                             outputs=("logp", "entropy", "dlogp", "lse", "lse64"), **kw)
        obj.merge_gradients(cfg)
        obj.sync()
    # fused update pass (fp32 cluster kernel) + backward epilogue
    V = 32000
    toks = t(rng.integers(0, V, (B, T)).astype(np.int32))
    L = [logits(B * T, V, torch.float32, model=m) for m in range(3)]
    adv = t(rng.uniform(-1, 1, (B, T)).astype(np.float32))
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k2", loss_agg="seq-mean-token-mean", group_size=2)
    cnt = obj.batch_counts(cfg, lengths, T, mask=mask)
    w = obj.loss_weights(cfg, lengths, cnt, T, mask=mask)
    outs = obj.ppo_gradient(cfg, toks, lengths, L[0], adv, mask=mask, old_logits=L[1], ref_logits=L[2],
                            outputs=("dlogp", "lse", "lse64"))
    obj.merge_gradients(cfg)
    obj.logits_backward(toks, lengths, L[0], outs["lse"], outs["dlogp"], w)
    obj.logits_backward(toks, lengths, L[0], outs["lse64"], outs["dlogp"], w)
    for gdt in (torch.float32, torch.bfloat16):
        obj.ppo_gradient_fused(cfg, toks, lengths, L[0], adv, w, mask=mask, old_logits=L[1], ref_logits=L[2],
                               grad_dtype=gdt)
        obj.merge_gradients(cfg)
    os.environ["RLO_FUSED_SLICE_KB"] = "40"  # forced bf16 8-CTA cluster (read at handle creation)
    objf = rlo.Objective(0)
    del os.environ["RLO_FUSED_SLICE_KB"]
    Vq = 152064
    Lb = [logits(B * T, Vq, torch.bfloat16, model=m) for m in range(3)]
    toksq = t(rng.integers(0, Vq, (B, T)).astype(np.int32))
    wq = objf.loss_weights(cfg, lengths, objf.batch_counts(cfg, lengths, T, mask=mask), T, mask=mask)
    objf.ppo_gradient_fused(cfg, toksq, lengths, Lb[0], adv, wq, mask=mask, old_logits=Lb[1], ref_logits=Lb[2],
                            grad_dtype=torch.bfloat16)
    objf.merge_gradients(cfg)
    # advantages: REINFORCE / GAE scans and GRPO, whitening on and off
    Bg, Tg = 8, 37
    lg = rng.integers(0, Tg + 1, Bg).astype(np.int32)
    lg[0] = Tg
    Lg = t(lg)
    mg = (rng.random((Bg, Tg)) < 0.7).astype(np.uint8)
    mg[0, 0] = 1
    Mg = t(mg)
    rw = t(rng.standard_normal((Bg, Tg)).astype(np.float32))
    vals = t(rng.standard_normal((Bg, Tg)).astype(np.float32))
    rs = t(rng.integers(0, 2, Bg).astype(np.float32))
    for est in ("reinforce", "gae", "grpo"):
        for wh in (False, True):
            c = rlo.TrainConfig(adv_estimator=est, whiten_advantages=wh, group_size=4, gamma=0.99)
            obj.compute_advantages(c, Lg, T=Tg, mask=Mg, rewards=None if est == "grpo" else rw,
                                   scalar_rewards=rs if est == "grpo" else None,
                                   values=vals if est == "gae" else None, returns=True)
    # device-side merge (graph-capturable step) and value loss
    obj.ppo_gradient(cfg, toks, lengths, L[0], adv, old_logits=L[1], ref_logits=L[2])
    buf = obj.merge_gradients_async(cfg)
    rlo.Objective.step_result(buf)
    obj.value_loss(Lg, vals, rw, old_values=vals * 0.9, value_clip=0.2, mask=Mg)
    # decode: screen + fp64 redo, two vocabularies, several temperatures
    for dt, Vd in ((torch.bfloat16, 152064), (torch.float32, 4099)):
        x = logits(16, Vd, dt)
        keys = t(rng.integers(0, 2**62, 16).astype(np.int64))
        pos = t(np.arange(16, dtype=np.int64))
        for temp in (1.0, 0.7, 1e-7):
            obj.decode_sample(x, temp, 5, 1, keys, pos)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
