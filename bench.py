#!/usr/bin/env python3
"""Benchmark of the B200 RL-objective path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

One step = one pass of the whole hot path over one batch: advantages
(REINFORCE/GRPO/GAE + clipping/whitening) -> fused vocab pass over the actor,
old-policy and reference logits (log-probs, entropy, KL, clipped/dual-clipped
surrogate, dlogp) -> deterministic merge (UpdateStats).  Logits are
synthetic (include/rlo_synth.h) and resident in HBM; configs whose logits do
not fit stream micro-batches of whole groups through a resident chunk (each
row still read from HBM).  Multi-GPU: one process per GPU (torchrun), each
rank owns its own batch of the config's size (weak scaling); NCCL carries only
the global whitening statistics and the loss-normalisation partials.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))

if int(os.environ.get("WORLD_SIZE", "1")) > 1 and os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    # NCCL's communicator-init lines (rank, nranks, NVLink / NVLS topology) go to
    # stderr with an N > 1 run, so a scaling record can confirm the group it ran
    # on; set before torch loads NCCL, which reads the level once
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
sys.path.insert(0, ROOT)

METRIC = "scored tokens/sec (logprob+KL+adv+PPO loss); HBM GB/s vs peak; 1/2/4/8 GPU"

# BASELINE.json configs (index 1..5)
CONFIGS = {
    1: dict(name="cfg1: GRPO 64 prompts x 8 responses x 512 tokens, V=32000 fp32 logits, token-mean",
            B=512, T=512, V=32000, dtype="f32", est="grpo", G=8, whiten=False, kl_est="k1", kl_coef=0.0,
            dual=0.0, agg="token-mean", mb_seqs=None),
    2: dict(name="cfg2: PPO+GAE (gamma=1, lambda=0.95) + k3 KL vs ref, 256 seqs x 1024 tokens, V=32000 fp32 logits",
            B=256, T=1024, V=32000, dtype="f32", est="gae", G=1, whiten=True, kl_est="k3", kl_coef=0.01,
            dual=0.0, agg="token-mean", mb_seqs=None),
    3: dict(name="cfg3: GRPO 128 prompts x 16 responses x 2048 tokens, V=152064 bf16 logits, token-mean",
            B=2048, T=2048, V=152064, dtype="bf16", est="grpo", G=16, whiten=False, kl_est="k3", kl_coef=0.001,
            dual=0.0, agg="token-mean", mb_seqs=16),
    4: dict(name="cfg4: long-CoT RLVR 32 prompts x 8 responses x 16384 tokens, V=152064 bf16, dual-clip c=3, "
                 "global whitening", B=256, T=16384, V=152064, dtype="bf16", est="grpo", G=8, whiten=True,
            kl_est="k3", kl_coef=0.001, dual=3.0, agg="token-mean", mb_seqs=2),
    5: dict(name="cfg5: GRPO 1024 prompts x 8 responses x 4096 tokens, V=152064 bf16, global whitening, "
                 "global batch sharded over the GPUs",
            B=8192, T=4096, V=152064, dtype="bf16", est="grpo", G=8, whiten=True, kl_est="k3", kl_coef=0.001,
            dual=0.0, agg="token-mean", mb_seqs=8, global_batch=True),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clocks + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index, period=0.01):
        self.index, self.period = index, period
        self.samples, self.reasons, self.power = [], set(), []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:
                self.limit_w = None
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w": statistics.median(self.power) if self.power else None, "power_limit_w": self.limit_w}


def make_cfg(rlo, c):
    return rlo.TrainConfig(adv_estimator=c["est"], group_size=c["G"], whiten_advantages=c["whiten"],
                           kl_estimator=c["kl_est"], kl_coef=c["kl_coef"], dual_clip_c=c["dual"], loss_agg=c["agg"],
                           gamma=1.0, lambd=0.95, clip_eps=0.2, advantage_clip=10.0, reward_clip=20.0)


def side_inputs(c, rank, seed):
    """Per-rank synthetic SampleBatch side arrays (host numpy).  Global-batch
    configs draw the whole batch from one seed and keep this rank's shard."""
    B, T = c["B"], c["T"]
    if c.get("global_batch"):
        full = side_inputs(dict(c, B=c["B_global"], global_batch=False), 0, seed)
        return {k: v[c["b0"]:c["b0"] + B] for k, v in full.items()}
    rng = np.random.default_rng(seed * 1000 + rank)
    lengths = np.full(B, T, np.int32)  # throughput runs: full-length responses
    if c["est"] == "grpo":
        p = np.repeat(rng.uniform(0.1, 0.9, B // c["G"]), c["G"])
        rs = (rng.random(B) < p).astype(np.float32)  # binary accuracy reward (rewards.cpp:463-468)
        return dict(lengths=lengths, scalar_rewards=rs)
    rt = np.zeros((B, T), np.float32)
    rt[:, -1] = rng.uniform(-1, 1, B)
    rt[rng.random(B) < 0.05, -1] = 30.0  # exercises reward_clip
    vals = (rng.standard_normal((B, T)) * 0.5).astype(np.float32)
    return dict(lengths=lengths, rewards=rt, values=vals)


def run_ours(args, c):
    import torch

    import paper_2506_06122_b200 as rlo

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    obj = rlo.Objective(local)
    if world > 1:
        uid = [rlo.Objective.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        obj.init_comm(uid[0], rank, world)

    if c.get("global_batch"):
        # batch-sharded (BASELINE cfg 5): the global batch is split on group
        # boundaries (rlo_shard_plan, the reference's split rule over groups)
        b0, nb = rlo.shard_plan(c["B"], c["G"], world, rank)
        c = dict(c, B_global=c["B"], B=nb, b0=b0)
    B, T, V = c["B"], c["T"], c["V"]
    tdt = torch.float32 if c["dtype"] == "f32" else torch.bfloat16
    esz = 4 if c["dtype"] == "f32" else 2
    mb = c["mb_seqs"] or B
    key_rows = mb * T
    seed = args.seed
    row_off = (c["b0"] if c.get("global_batch") else rank * B) * T
    stream = torch.cuda.current_stream(dev)

    # resident logits: all rows, or one micro-batch chunk reused by every micro-batch
    logits = [torch.empty(key_rows, V, dtype=tdt, device=dev) for _ in range(3)]
    for m in range(3):
        rlo.synth_logits(logits[m], seed=seed, model=m, row_key_offset=row_off)
    tokens = torch.empty(B, T, dtype=torch.int32, device=dev)
    rlo.synth_tokens(tokens, V, seed=seed, row_key_offset=row_off, key_rows=key_rows)
    side = side_inputs(c, rank, seed)
    dside = {k: torch.from_numpy(v).to(dev) for k, v in side.items()}
    cfg = make_cfg(rlo, c)
    adv = torch.empty(B, T, dtype=torch.float32, device=dev)
    logp = torch.empty(B, T, dtype=torch.float32, device=dev)
    nmb = B // mb
    torch.cuda.synchronize()

    vocab_ms = []
    record = {"on": False}

    def step():
        obj.compute_advantages(cfg, dside["lengths"], T=T, rewards=dside.get("rewards"),
                               scalar_rewards=dside.get("scalar_rewards"), values=dside.get("values"), out=adv)
        for i in range(nmb):
            s = slice(i * mb, (i + 1) * mb)
            if record["on"]:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            _ppo(obj, rlo, cfg, tokens[s], dside["lengths"][s], logits, adv[s], i * mb, logp[s])
            if record["on"]:
                e1.record(stream)
                vocab_ms.append((e0, e1))
        return obj.merge_gradients(cfg)

    for _ in range(args.warmup):
        st = step()

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    n0 = rlo.launch_count()
    record["on"] = True
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            st = step()
        t1.record(stream)
        barrier()
    record["on"] = False
    launches = rlo.launch_count() - n0
    ms = t0.elapsed_time(t1)
    vk = [a.elapsed_time(b) for a, b in vocab_ms]
    vocab_avg_ms = float(np.mean(vk))
    vocab_avg_ms_slowest = vocab_avg_ms
    if dist:
        tt = torch.tensor([ms, vocab_avg_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, vocab_avg_ms_slowest = float(tt[0].item()), float(tt[1].item())

    nrow = B * T  # sampled results of the last timed step (checked in the CPU leg)
    sample_rows = sorted({0, nrow - 1, key_rows - 1, min(key_rows, nrow - 1), nrow // 2, (7 * nrow) // 11,
                          12345 % nrow})
    lp_sample = logp.view(-1)[torch.tensor(sample_rows, device=dev)].cpu().numpy()
    tok_sample = tokens.view(-1)[torch.tensor(sample_rows, device=dev)].cpu().numpy()

    # ---- P=1: actor-only pass, old/ref log-probs precomputed ----
    p1 = None if args.no_p1 else run_p1(args, c, obj, rlo, torch, cfg, logits, tokens, dside, adv, logp, stream,
                                       barrier, dist, mb, esz)

    # ---- e2e: the reference-facing host-buffer call ------------------------
    e2e = None if args.no_e2e else run_e2e(args, c, obj, rlo, torch, cfg, logits, side, dev, stream, dist,
                                           key_rows, mb)

    peak, peak_kind = load_peaks()
    traffic = traffic_from_profile(args.config)
    tokens_per_step = B * T  # full-length responses, all positions loss-participating
    per_row_side = 4 + 4 + 17  # token id, advantage, per-token results written for the reduction
    bytes_per_launch = mb * T * (3 * V * esz + per_row_side)
    achieved = bytes_per_launch / (vocab_avg_ms * 1e-3) / 1e9
    job_tokens = c.get("B_global", world * B) * T  # all ranks' scored tokens per step
    value = job_tokens * args.steps / (ms * 1e-3)

    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if c.get("global_batch") else "weak",
        "vs_baseline": None, "dtype": c["dtype"],
        "data": "synthetic: counter-hash logits (include/rlo_synth.h), random-init side arrays",
        "config": {"workload": c["name"], "B_per_rank": B, "T": T, "V": V, "logits_tensors": 3,
                   "global_batch_seqs": c.get("B_global", B * world), "micro_batch_seqs": mb,
                   "resident_logit_rows": key_rows,
                   "l2": f"inputs larger than L2: {3 * key_rows * V * esz / 1e9:.1f} GB of logits streamed per "
                         f"micro-batch vs 126 MB L2",
                   "parallelism": f"dp{world}"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic[0], "traffic_source": traffic[1], "peak_kind": peak_kind,
                     "frac_of_spec_8000": achieved / 8000.0,
                     "kernel": "vocab_kernel (fused 3-tensor logprob+entropy+loss pass, incl. per-seq reduce)",
                     "bytes_per_launch": bytes_per_launch, "avg_launch_ms": vocab_avg_ms,
                     **({"avg_launch_ms_slowest_rank": vocab_avg_ms_slowest} if world > 1 else {})},
        "e2e": e2e,
        "p1": p1,
        "gpu_launches": launches,
        "clocks": clk.result(),
        "stats": {"loss": st.loss, "mean_ratio": st.mean_ratio, "clip_fraction": st.clip_fraction,
                  "mean_kl": st.mean_kl, "tokens": st.tokens, "mean_entropy": st.mean_entropy},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the last timed step's actor log-probs on a few sampled token rows, for
        # the oracle check inside the CPU leg (row r reads resident logits row
        # r mod key_rows; rank 0: token and logits keys coincide)
        out["cpu_baseline"] = cpu_baseline(args, c, target_s=args.cpu_seconds,
                                           check=(sample_rows, key_rows, lp_sample, tok_sample))
    obj.close()
    if dist:
        dist.destroy_process_group()
    return out if rank == 0 else None


def _ppo(obj, rlo, cfg, tokens, lengths, logits, adv, seq_offset, logp, old_lp=None, ref_lp=None):
    """One fused vocab pass: logits = [actor, old, ref] (P=3) or [actor] with
    precomputed old/ref log-probs (P=1)."""
    import ctypes as C

    from paper_2506_06122_b200 import _abi
    from paper_2506_06122_b200.errors import check
    from paper_2506_06122_b200.policy import _batch, _logits, _stream
    o = _abi.rlo_token_out()
    o.logp = logp.data_ptr()
    L = [_logits(x) for x in logits]
    vp = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    check(_abi.lib().rlo_ppo_gradient(obj._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, tokens, None,
                                                                                    tokens.shape[1], seq_offset)),
                                      C.byref(L[0]), C.byref(L[1]) if len(L) > 1 else None,
                                      C.byref(L[2]) if len(L) > 2 else None, vp(old_lp), vp(ref_lp),
                                      C.c_void_p(adv.data_ptr()), C.byref(o), _stream(None, logp.device)))


def run_p1(args, c, obj, rlo, torch, cfg, logits, tokens, dside, adv, logp, stream, barrier, dist, mb, esz):
    """The reference pipeline's shape: old log-probs come from sampling time
    (policy.cpp:356) and ref log-probs from a separate pass (pipeline.cpp:508),
    so the update reads only the actor logits (P=1).  old/ref log-probs are
    computed once here (untimed) with forward_logprobs."""
    B, T, V = c["B"], c["T"], c["V"]
    old_lp = torch.empty(B, T, dtype=torch.float32, device=tokens.device)
    ref_lp = torch.empty_like(old_lp)
    for i in range(B // mb):
        s = slice(i * mb, (i + 1) * mb)
        old_lp[s] = obj.forward_logprobs(logits[1], tokens[s], dside["lengths"][s])["logp"]
        ref_lp[s] = obj.forward_logprobs(logits[2], tokens[s], dside["lengths"][s])["logp"]
    ev = []

    def step(rec):
        obj.compute_advantages(cfg, dside["lengths"], T=T, rewards=dside.get("rewards"),
                               scalar_rewards=dside.get("scalar_rewards"), values=dside.get("values"), out=adv)
        for i in range(B // mb):
            s = slice(i * mb, (i + 1) * mb)
            if rec:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            _ppo(obj, rlo, cfg, tokens[s], dside["lengths"][s], logits[:1], adv[s], i * mb, logp[s],
                 old_lp[s], ref_lp[s])
            if rec:
                e1.record(stream)
                ev.append((e0, e1))
        return obj.merge_gradients(cfg)

    for _ in range(args.warmup):
        step(False)
    steps = args.steps
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        st = step(True)
    t1.record(stream)
    barrier()
    ms = t0.elapsed_time(t1)
    if dist:
        tt = torch.tensor([ms], device=tokens.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    world = dist.get_world_size() if dist else 1
    job_tokens = c.get("B_global", world * B) * T
    vk = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    bytes_per_launch = mb * T * (V * esz + 4 + 4 + 8 + 17)
    peak, _ = load_peaks()
    return {"value": job_tokens * steps / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms / steps,
            "logits_tensors": 1, "achieved_gbs": bytes_per_launch / (vk * 1e-3) / 1e9,
            "frac": bytes_per_launch / (vk * 1e-3) / 1e9 / peak, "avg_launch_ms": vk,
            "loss": st.loss, "note": "actor logits only; old/ref log-probs precomputed (untimed)"}


def run_e2e(args, c, obj, rlo, torch, cfg, logits, side, dev, stream, dist, key_rows, mb):
    """Same metric through the public host-buffer API: per step the SampleBatch
    arrays are copied H2D from pinned memory and advantages + actor log-probs
    (and UpdateStats) come back D2H.  Logits stay device-resident: they are the
    model forward's on-device output, not a host input."""
    B, T, V = c["B"], c["T"], c["V"]
    pin = {k: torch.from_numpy(v).pin_memory() for k, v in side.items()}
    tok_host = torch.empty(B, T, dtype=torch.int32).pin_memory()
    rlo.synth_tokens(tok_host_dev := torch.empty(B, T, dtype=torch.int32, device=dev), V, seed=args.seed,
                     row_key_offset=c.get("b0", int(os.environ.get("RANK", "0")) * B) * T, key_rows=key_rows)
    tok_host.copy_(tok_host_dev)
    adv_host = torch.empty(B, T, dtype=torch.float32).pin_memory()
    logp_host = torch.empty(B, T, dtype=torch.float32).pin_memory()
    hb_in = sum(v.numel() * v.element_size() for v in pin.values()) + tok_host.numel() * 4
    hb_out = 2 * B * T * 4

    if mb == B:
        def step():
            return obj.step_host(cfg, tok_host.numpy(), pin["lengths"].numpy(), logits[0],
                                 rewards=pin["rewards"].numpy() if "rewards" in pin else None,
                                 scalar_rewards=pin["scalar_rewards"].numpy() if "scalar_rewards" in pin else None,
                                 values=pin["values"].numpy() if "values" in pin else None, old_logits=logits[1],
                                 ref_logits=logits[2], adv_out=adv_host.numpy(), logp_out=logp_host.numpy())
        api = "rlo_objective_step_host (C ABI, host buffers)"
    else:
        # micro-batched: the whole batch's host arrays go in once, the logits
        # callback names each micro-batch's device logits (here the resident
        # chunk, which a trainer's model forward would refill), results come back
        def logits_fn(i, b0, nb):
            return logits[0], logits[1], logits[2]

        def step():
            return obj.step_host_mb(cfg, tok_host.numpy(), pin["lengths"].numpy(), mb, logits_fn,
                                    rewards=pin["rewards"].numpy() if "rewards" in pin else None,
                                    scalar_rewards=pin["scalar_rewards"].numpy() if "scalar_rewards" in pin else None,
                                    values=pin["values"].numpy() if "values" in pin else None,
                                    adv_out=adv_host.numpy(), logp_out=logp_host.numpy())
        api = "rlo_objective_step_host_mb (C ABI, host buffers, per-micro-batch logits callback)"

    for _ in range(max(1, args.warmup)):
        step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist:
        tt = torch.tensor([el], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    world = dist.get_world_size() if dist else 1
    return {"value": c.get("B_global", world * B) * T * args.steps / el, "unit": "tokens/s", "h2d_bytes_per_step": hb_in,
            "d2h_bytes_per_step": hb_out + 64, "api": api, "ms_per_step": 1e3 * el / args.steps}


def kernel_sig(name):
    """Normalised template signature of a vocab_ldg_kernel instantiation from
    an ncu or c++filt kernel name: 'vocab_ldg_kernel<32,__nv_bfloat16,3,...>'
    (bools as 0 / 1, no spaces)."""
    import re
    m = re.search(r"vocab_ldg_kernel<[^()]*>", name)
    if not m:
        return None
    sig = m.group(0).replace(" ", "").replace("true", "1").replace("false", "0")
    return sig.replace("(anonymousnamespace)::", "")


def kernel_sass_hash(lib=None, sig=None):
    """sha256 of the SASS of one vocab-pass kernel instantiation (`sig`, see
    kernel_sig; every vocab_ldg_kernel instantiation when None) in the
    library this run loaded (cuobjdump -sass, addresses stripped): identifies
    the kernel a stored ncu capture was taken from, independent of host code,
    comments or changes to other kernels."""
    import hashlib
    import re
    import subprocess
    from paper_2506_06122_b200 import _abi
    lib = lib or _abi.LIB_PATH
    try:
        out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, timeout=120).stdout
        names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function : (\S+)", out)),
                               capture_output=True, text=True, timeout=60).stdout.splitlines()
    except Exception:
        return None
    demangled = dict(zip(re.findall(r"Function : (\S+)", out), names))
    keep, lines = False, []
    for ln in out.splitlines():
        if "Function :" in ln:
            fn = demangled.get(ln.split("Function :")[1].strip(), "")
            keep = "vocab_ldg_kernel" in fn and (sig is None or kernel_sig(fn) == sig)
        if keep and ("Function :" in ln or re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln)):
            lines.append(re.sub(r"/\*[0-9a-f]{4,}\*/|/\* 0x[0-9a-f]+ \*/", "", ln).strip())
    if not lines:
        return None
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()[:16]


def traffic_from_profile(cfg_id):
    """DRAM bytes per launch of the vocab kernel from the committed ncu
    capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py) --
    used only when that capture was taken from the very kernels this run
    loaded (SASS hash match); otherwise null, never a stale value."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, "no capture"
    with open(p) as f:
        d = json.load(f)
    v = d.get(f"cfg{cfg_id}")
    if v is None:
        return None, "no capture for this config"
    if v.get("sass_hash") is None or v.get("sass_hash") != kernel_sass_hash(sig=v.get("kernel_sig")):
        return None, "capture is from another build of this kernel (SASS hash differs: stale): not used"
    return v.get("bytes_per_launch"), f"ncu capture {v.get('capture', '')} (kernel SASS {v.get('sass_hash')})"


def oracle_check(O, c, seed, check):
    """The timed run's own results against the fp64 oracle: actor log-probs of
    sampled token rows of the last timed step (|gpu - oracle| <= 1e-5 *
    max(1, |oracle|), the north_star tolerance)."""
    rows, key_rows, lp_gpu, toks = check
    dt = O.F32 if c["dtype"] == "f32" else O.BF16
    worst = 0.0
    for r, g, tok in zip(rows, lp_gpu, toks):
        z = O.synth_row(dt, c["V"], seed, 0, r % key_rows)
        lse, _ = O.logsoftmax_row(z)
        want = z[int(tok)] - lse
        worst = max(worst, abs(float(g) - want) / max(1.0, abs(want)))
    return {"rows": len(rows), "what": "actor logp of sampled rows of the last timed step vs oracle",
            "max_scaled_err": float(worst), "tol": 1e-5, "ok": bool(worst <= 1e-5)}


def cpu_baseline(args, c, target_s=12.0, use_ref=None, check=None):
    """The reference's CPU path (oracle/_ref: the reference's own
    next_token_forward log-softmax, compute_advantages, merge_gradients) on a
    bounded sample of the same workload, all host threads.  With `check`, the
    GPU run's sampled results are first checked against the oracle."""
    import oracle as O
    chk_out = oracle_check(O, c, args.seed, check) if check is not None else None
    if use_ref is None:
        use_ref = O.ref_available()
    threads = os.cpu_count() or 1
    oc = O.TrainConfig(adv_estimator={"reinforce": 0, "grpo": 1, "gae": 2}[c["est"]], group_size=c["G"],
                       whiten_advantages=int(c["whiten"]), kl_estimator={"k1": 0, "k2": 1, "k3": 2}[c["kl_est"]],
                       kl_coef=c["kl_coef"], dual_clip_c=c["dual"])
    dt = O.F32 if c["dtype"] == "f32" else O.BF16
    T, V, G = c["T"], c["V"], c["G"]
    key_rows = 256
    # calibrate: one sequence-slice per thread
    Tc = max(8, min(T, 64))
    Bc = max(G, ((threads + G - 1) // G) * G)
    secs, _ = O.bench_objective(threads, oc, dt, V, Bc, Tc, key_rows, args.seed, use_ref=use_ref)
    rate = Bc * Tc / max(secs, 1e-9)
    want_tokens = max(Bc * Tc, int(rate * target_s))
    Bs = max(Bc, min(c["B"], (want_tokens // T // G) * G))
    Ts = T if Bs * T <= want_tokens * 2 else max(8, want_tokens // Bs)
    secs, chk = O.bench_objective(threads, oc, dt, V, Bs, Ts, key_rows, args.seed, use_ref=use_ref)
    return {"value": Bs * Ts / secs, "unit": "tokens/s", "cores": threads,
            "kind": "reference" if use_ref else "port",
            "sample": f"{Bs} seqs x {Ts} tokens of {c['name'].split(':')[0]} (V={V} {c['dtype']}, 3 logits "
                      f"passes via the reference's next_token_forward log-softmax, {key_rows} resident rows/model), "
                      f"{secs:.1f} s", "seconds": secs, "checksum_loss": chk, "B_sample": Bs, "T_sample": Ts,
            **({"gpu_oracle_check": chk_out} if chk_out is not None else {})}


def run_reference(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O
    use_ref = O.ref_available()
    per_step = max(1.0, args.ref_step_seconds)
    base = cpu_baseline(args, c, target_s=per_step, use_ref=use_ref)
    Bs, Ts = base["B_sample"], base["T_sample"]
    oc = O.TrainConfig(adv_estimator={"reinforce": 0, "grpo": 1, "gae": 2}[c["est"]], group_size=c["G"],
                       whiten_advantages=int(c["whiten"]), kl_estimator={"k1": 0, "k2": 1, "k3": 2}[c["kl_est"]],
                       kl_coef=c["kl_coef"], dual_clip_c=c["dual"])
    dt = O.F32 if c["dtype"] == "f32" else O.BF16
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        O.bench_objective(threads, oc, dt, c["V"], Bs, Ts, 256, args.seed, use_ref=use_ref)
    tot = 0.0
    for _ in range(args.steps):
        s, _ = O.bench_objective(threads, oc, dt, c["V"], Bs, Ts, 256, args.seed, use_ref=use_ref)
        tot += s
    value = Bs * Ts * args.steps / tot
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": 0,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: counter-hash logits (include/rlo_synth.h)",
           "config": {"workload": c["name"], "B_per_rank": c["B"], "T": c["T"], "V": c["V"], "logits_tensors": 3},
           "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads,
                            "kind": "reference" if use_ref else "port", "sample": base["sample"]},
           "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS),
                    help="BASELINE.json config (default 3: the north_star's Qwen2.5-7B-vocab bf16 batch)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-p1", action="store_true", help="skip the actor-only (P=1) leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    c = CONFIGS[args.config]
    # stdout carries exactly one JSON line: anything libraries print (NCCL's
    # version banner, warnings) is routed to stderr while the run executes.
    sys.stdout.flush()
    real_stdout = os.dup(1)
    os.dup2(2, 1)
    try:
        out = run_reference(args, c) if args.impl == "reference" else run_ours(args, c)
    finally:
        sys.stdout.flush()
        os.dup2(real_stdout, 1)
        os.close(real_stdout)
    if out is not None:
        print(json.dumps(out), flush=True)
    # exit-time library output (NCCL's plugin teardown prints INFO lines at
    # process exit under NCCL_DEBUG=INFO) goes to stderr, after the one line
    os.dup2(2, 1)


if __name__ == "__main__":
    main()
