"""Measurements of the SURVEY.md §8f rows around the path (one JSON line each):

  decode     sampling-time log-probs (rlo_decode_sample, decode_next policy.cpp:143-169):
             rows/s and the HBM rate of one pass over each row
  value      critic value loss (rlo_value_loss, value_gradient policy.cpp:474-540): tokens/s
  jsonl      SampleBatch JSONL ingestion (rlo_batch_from_jsonl) against the reference's own
             SampleBatch::from_jsonl + validate (oracle/_ref, when built): MB/s of JSONL
  broadcast  ModelUpdateGroup bucketed NCCL broadcast (rlo_broadcast_params), under torchrun
             with >= 2 ranks: algorithm bandwidth per bucket size
  reference  the reference's own CPU code for decode / actor backward / value / advantages
             (oracle/_ref, cpu_baseline role) on all host threads, bounded samples

The actor backward epilogue (row 1) is measured by tools/bench_update.py.

    python tools/bench_next.py [--only decode,value,jsonl]
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/bench_next.py --only broadcast
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_06122_b200 as rlo  # noqa: E402


def timed(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def bench_decode(obj):
    for rows, V, dt, stride in ((4096, 152064, torch.bfloat16, 152064), (32768, 152064, torch.bfloat16, 152064),
                                (32768, 32000, torch.float32, 32000), (32768, 50257, torch.bfloat16, 50257),
                                (32768, 50257, torch.bfloat16, 50264)):
        x = torch.empty(rows, stride, dtype=dt, device="cuda")[:, :V]
        rlo.synth_logits(x, seed=1, model=0)
        keys = torch.arange(rows, dtype=torch.int64, device="cuda") * 7919
        pos = torch.full((rows,), 17, dtype=torch.int64, device="cuda")
        byts = rows * V * x.element_size()
        for temp in (0.8, 1.0):
            for margin in ("", "0"):  # screened fp32 path (default) / fp64 path only
                os.environ["RLO_DECODE_MARGIN"] = margin
                o = rlo.Objective(obj.device)  # knobs are read when a handle is created
                ms = timed(lambda: o.decode_sample(x, temp, 42, 3, keys, pos))
                print(json.dumps({"row": "decode", "rows": rows, "V": V, "stride": stride,
                                  "dtype": str(dt).split(".")[-1], "temperature": temp,
                                  "path": "fp64" if margin == "0" else "screened", "ms": ms,
                                  "rows_per_s": rows / ms * 1e3, "gbs_one_pass": byts / ms / 1e6,
                                  "note": "bytes = one pass over each row"}), flush=True)
        os.environ.pop("RLO_DECODE_MARGIN", None)
        del x


def bench_value(obj):
    B, T = 256, 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    v = torch.randn(B, T, device="cuda", generator=g)
    vo = v + 0.1 * torch.randn(B, T, device="cuda", generator=g)
    R = torch.randn(B, T, device="cuda", generator=g)
    L = torch.full((B,), T, dtype=torch.int32, device="cuda")
    ms = timed(lambda: obj.value_loss(L, v, R, old_values=vo, value_clip=0.2))
    byts = B * T * (4 * 3 + 4)
    print(json.dumps({"row": "value", "B": B, "T": T, "ms": ms, "tokens_per_s": B * T / ms * 1e3,
                      "gbs": byts / ms / 1e6, "note": "includes the host sync of the stats"}), flush=True)


def _big_jsonl(n, T, seed=5):
    """A rollout batch the size the path consumes: n samples x T tokens with
    old / ref log-probs (the reference's record keys, sample.cpp:124-140)."""
    rng = np.random.default_rng(seed)
    lines = []
    for i in range(n):
        toks = rng.integers(0, 152064, T)
        lp = np.round(rng.uniform(-8, 0, T), 6)
        ref = np.round(lp + rng.uniform(-0.1, 0.1, T), 6)
        lines.append(json.dumps({"sample_id": f"s{i}", "group_id": f"g{i // 8}",
                                 "response_tokens": toks.tolist(), "response_logprobs": lp.tolist(),
                                 "ref_logprobs": ref.tolist(), "scalar_reward": float(rng.random() < 0.5)}))
    return "\n".join(lines)


def bench_advantages(obj):
    """compute_advantages at long-CoT shapes (the O(N) part of the path)."""
    for est, B, T in (("gae", 256, 16384), ("gae", 2048, 2048), ("reinforce", 256, 16384), ("grpo", 2048, 2048)):
        g = torch.Generator(device="cuda").manual_seed(1)
        L = torch.full((B,), T, dtype=torch.int32, device="cuda")
        kw = {}
        if est == "grpo":
            kw["scalar_rewards"] = torch.rand(B, device="cuda", generator=g)
        else:
            kw["rewards"] = torch.randn(B, T, device="cuda", generator=g) * 0.1
        if est == "gae":
            kw["values"] = torch.randn(B, T, device="cuda", generator=g) * 0.5
        cfg = rlo.TrainConfig(adv_estimator=est, group_size=16 if est == "grpo" else 1, whiten_advantages=True,
                              gamma=0.99, lambd=0.95)
        out = torch.empty(B, T, device="cuda")
        ms = timed(lambda: obj.compute_advantages(cfg, L, T=T, out=out, **kw))
        byts = B * T * (4 + 4 + (4 if est == "gae" else 0) + 8 + 8)  # rewards, adv, values, fp64 scratch w+r
        print(json.dumps({"row": "advantages", "estimator": est, "B": B, "T": T, "ms": ms,
                          "tokens_per_s": B * T / ms * 1e3, "gbs": byts / ms / 1e6,
                          "note": "whitened (global stats), fp64 scan"}), flush=True)


def bench_jsonl():
    import oracle as O
    cases = []
    if O.ref_available():
        cases.append(("reference SampleBatch::to_jsonl, 512 samples", O.ref_batch_jsonl(5, 512)))
    cases.append(("synthetic 2048 samples x 1024 tokens", _big_jsonl(2048, 1024)))
    for src, text in cases:
        mb = len(text.encode()) / 1e6
        data = text.encode()

        def timeit(fn, budget=2.0):
            t0, k = time.perf_counter(), 0
            while k < 1 or time.perf_counter() - t0 < budget:
                fn()
                k += 1
            return (time.perf_counter() - t0) / k
        ours = timeit(lambda: rlo.batch_from_jsonl(data))
        os.environ["RLO_JSONL_THREADS"] = "1"
        serial = timeit(lambda: rlo.batch_from_jsonl(data))
        del os.environ["RLO_JSONL_THREADS"]
        out = {"row": "jsonl", "source": src, "mb": round(mb, 2), "ms": ours * 1e3, "mb_per_s": mb / ours,
               "threads": os.cpu_count(), "serial_mb_per_s": mb / serial}
        if O.ref_available():
            ref = timeit(lambda: O.ref_parse_validate_jsonl(text))
            out.update(reference_ms=ref * 1e3, reference_mb_per_s=mb / ref, speedup=ref / ours)
        print(json.dumps(out), flush=True)


def bench_reference():
    """The reference's own CPU code for the same rows (oracle/_ref, the
    cpu_baseline role: timed beside the GPU numbers, never the product), on
    all host threads over a bounded sample: ctypes drops the GIL inside each
    call, so one Python thread per core runs the reference's functions in
    parallel like the reference's thread-per-rank cluster."""
    import concurrent.futures as cf

    import oracle as O
    if not O.ref_available():
        print(json.dumps({"row": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
        return
    nt = os.cpu_count() or 1
    pool = cf.ThreadPoolExecutor(nt)

    def par(fn, n, budget=1.5):
        """Rounds of n calls over the pool until `budget` seconds: (s, calls)."""
        t0, k = time.perf_counter(), 0
        while k == 0 or time.perf_counter() - t0 < budget:
            list(pool.map(fn, range(k * n, (k + 1) * n)))
            k += 1
        return time.perf_counter() - t0, k * n

    V = 152064
    rng = np.random.default_rng(3)
    rows = [rng.standard_normal(V) * 3.0 for _ in range(nt)]
    for temp in (0.8, 1.0):  # decode_next (policy.cpp:143-169) on one logits row each
        s, n = par(lambda i: O.ref_decode_b2(rows[i % nt], temp, 42, 3, 7919 * i, 17), nt)
        print(json.dumps({"row": "decode", "impl": "reference", "V": V, "temperature": temp, "rows": n,
                          "threads": nt, "s": s, "rows_per_s": n / s}), flush=True)
    T = 8  # ppo_gradient incl. its actor backward dz = dlp (onehot - p) (policy.cpp:313-379), b2 trick
    lengths, mask = np.array([T], np.int32), np.ones(T, np.uint8)
    toks = rng.integers(0, V, T).astype(np.int32)
    lp = np.full(T, -3.0)
    adv = rng.uniform(-1, 1, T)
    cfg = O.TrainConfig(kl_coef=0.001)
    s, n = par(lambda i: O.ref_ppo_grad_b2(rows[i % nt], 1, T, lengths, toks, mask, lp, lp, adv, cfg), nt)
    print(json.dumps({"row": "backward", "impl": "reference", "V": V, "tokens": n * T, "threads": nt, "s": s,
                      "tokens_per_s": n * T / s, "note": "ppo_gradient: log-softmax + loss + dz per token"}),
          flush=True)
    B, T = 256, 16384  # value_gradient (policy.cpp:474-540) and compute_advantages (policy.cpp:257-311)
    L = np.full(B, T, np.int32)
    tg = rng.standard_normal(B * T)
    bt = B // nt or 1
    s, n = par(lambda i: O.ref_value_loss_b2(0.1, bt, T, L[:bt], None, tg[:bt * T]), nt)
    print(json.dumps({"row": "value", "impl": "reference", "B": B, "T": T, "threads": nt, "s": s,
                      "tokens_per_s": bt * n * T / s}), flush=True)
    acfg = O.TrainConfig(whiten_advantages=1, gamma=0.99)
    s, n = par(lambda i: O.ref_compute_advantages(acfg, bt, T, L[:bt], None, rewards_seq=np.ones(bt)), nt)
    print(json.dumps({"row": "advantages", "impl": "reference", "estimator": "reinforce", "B": B, "T": T,
                      "threads": nt, "s": s, "tokens_per_s": bt * n * T / s,
                      "note": "per-thread shards whitened locally (the reference has no GRPO/GAE)"}), flush=True)
    pool.shutdown()


def bench_broadcast():
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = rlo.Objective(local)
    uid = [rlo.Objective.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    obj.init_comm(uid[0], rank, world)
    buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB of parameters
    nbytes = buf.numel() * 4
    for bucket in (1 << 22, 1 << 26, 1 << 28, nbytes):
        dist.barrier()
        ms = timed(lambda: obj.broadcast_params(buf, bucket_bytes=bucket, root=0), iters=5, warm=2)
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"row": "broadcast", "world": world, "bytes": nbytes, "bucket_bytes": bucket,
                              "ms": float(t.item()), "algbw_gbs": nbytes / float(t.item()) / 1e6}), flush=True)
    obj.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="decode,value,advantages,jsonl,reference")
    args = ap.parse_args()
    rows = args.only.split(",")
    if "broadcast" in rows:
        bench_broadcast()
        return
    obj = rlo.Objective(0)
    if "decode" in rows:
        bench_decode(obj)
    if "value" in rows:
        bench_value(obj)
    if "advantages" in rows:
        bench_advantages(obj)
    if "jsonl" in rows:
        bench_jsonl()
    if "reference" in rows:
        bench_reference()


if __name__ == "__main__":
    main()
