"""Host-side mirror of the reference's RL-objective interface.

The reference (rollmini, proj/core) exposes the path as free functions in
``include/rollmini/policy.hpp``:

    forward_logprobs(params, batch)        policy.hpp:109  -> Objective.forward_logprobs
    compute_advantages(batch, config)      policy.hpp:118  -> Objective.compute_advantages
    ppo_gradient(params, batch, config)    policy.hpp:141  -> Objective.ppo_gradient
    merge_gradients(parts)                 policy.hpp:145  -> Objective.merge_gradients / merge_partials
    TrainConfig / UpdateStats              policy.hpp:57-67, 130-136

and behind the worker plugin ``Worker::call(method, Message)``
(worker.hpp:37-45; PolicyWorker policy_workers.cpp:46-64) -> ``PolicyWorker.call``.

The model forward is outside the path, so the B200 functions take the
model's logits (device tensors) where the reference takes ``PolicyParams``.
Every call goes through the C ABI of ``lib/librlo.so`` (sm_100a kernels);
torch is used only to hold device memory and to name the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _abi
from .errors import DispatchError, InputError, check

_ADV = {"reinforce": _abi.ADV_REINFORCE, "grpo": _abi.ADV_GRPO, "gae": _abi.ADV_GAE}
_KL = {"k1": _abi.KL_K1, "k2": _abi.KL_K2, "k3": _abi.KL_K3}
_AGG = {"token-mean": _abi.AGG_TOKEN_MEAN, "seq-mean-token-mean": _abi.AGG_SEQ_MEAN_TOKEN_MEAN,
        "seq-mean-token-sum": _abi.AGG_SEQ_MEAN_TOKEN_SUM, "group-mean": _abi.AGG_GROUP_MEAN}


@dataclass
class TrainConfig:
    """policy.hpp:57-67 (defaults :58-64, config keys config.cpp:197-205) + ROLL extensions."""

    clip_eps: float = 0.2
    kl_coef: float = 0.0
    learning_rate: float = 0.05
    advantage_clip: float = 10.0
    reward_clip: float = 20.0
    gamma: float = 1.0
    whiten_advantages: bool = False
    adv_estimator: str = "reinforce"
    lambd: float = 0.95
    kl_estimator: str = "k1"
    dual_clip_c: float = 0.0
    loss_agg: str = "token-mean"
    group_size: int = 1
    grpo_std_ddof: int = 0
    grpo_eps: float = 1e-6

    def to_c(self) -> _abi.rlo_train_config:
        c = _abi.rlo_train_config()
        c.clip_eps, c.kl_coef, c.learning_rate = self.clip_eps, self.kl_coef, self.learning_rate
        c.advantage_clip, c.reward_clip, c.gamma = self.advantage_clip, self.reward_clip, self.gamma
        c.whiten_advantages = int(bool(self.whiten_advantages))
        c.adv_estimator = _ADV[self.adv_estimator] if isinstance(self.adv_estimator, str) else int(self.adv_estimator)
        c.lambd = self.lambd
        c.kl_estimator = _KL[self.kl_estimator] if isinstance(self.kl_estimator, str) else int(self.kl_estimator)
        c.dual_clip_c = self.dual_clip_c
        c.loss_agg = _AGG[self.loss_agg] if isinstance(self.loss_agg, str) else int(self.loss_agg)
        c.group_size, c.grpo_std_ddof, c.grpo_eps = self.group_size, self.grpo_std_ddof, self.grpo_eps
        return c

    def validate(self) -> None:
        """TrainConfig::validate (policy.cpp:29-37), same messages, raises ConfigError."""
        check(_abi.lib().rlo_train_config_validate(C.byref(self.to_c())))


@dataclass
class UpdateStats:
    """policy.hpp:130-136 + extension stats."""

    loss: float = 0.0
    mean_ratio: float = 0.0
    clip_fraction: float = 0.0
    mean_kl: float = 0.0
    tokens: int = 0
    mean_entropy: float = 0.0
    dual_clip_fraction: float = 0.0
    seqs: int = 0
    groups: int = 0

    @classmethod
    def from_c(cls, s: _abi.rlo_stats) -> "UpdateStats":
        return cls(**{f.name: getattr(s, f.name) for f in fields(cls)})


def split_sizes(n: int, parts: int) -> list[int]:
    """sample.cpp:99-105 (contiguous, larger chunks first)."""
    out = (C.c_int64 * max(parts, 1))()
    check(_abi.lib().rlo_split_sizes(n, parts, out))
    return list(out[:parts])


def shard_plan(B: int, G: int, world: int, rank: int) -> tuple[int, int]:
    """Group-aligned data-parallel shard: (first sequence, count) of `rank`."""
    b, n = C.c_int32(), C.c_int32()
    check(_abi.lib().rlo_shard_plan(B, G, world, rank, C.byref(b), C.byref(n)))
    return b.value, n.value


def merge_partials(parts: np.ndarray, cfg: TrainConfig) -> UpdateStats:
    """merge_gradients scalar part (policy.cpp:421-450) over [nranks, 16] partials."""
    parts = np.ascontiguousarray(np.atleast_2d(parts), dtype=np.float64)
    arr = (_abi.rlo_partials * len(parts))()
    for i, p in enumerate(parts):
        arr[i].v[:] = p.tolist()
    st = _abi.rlo_stats()
    check(_abi.lib().rlo_merge_partials(arr, len(parts), C.byref(cfg.to_c()), C.byref(st)))
    return UpdateStats.from_c(st)


def whiten_combine(stats_all: np.ndarray):
    """(apply, mean, inv) from rank-ordered [world, 4] whitening statistics."""
    st = np.ascontiguousarray(np.atleast_2d(stats_all), dtype=np.float64)
    m, i = C.c_double(), C.c_double()
    ok = _abi.lib().rlo_whiten_combine(st.ctypes.data_as(C.c_void_p), st.shape[0], C.byref(m), C.byref(i))
    return bool(ok), m.value, i.value


def launch_count() -> int:
    return int(_abi.lib().rlo_launch_count())


# ---------------------------------------------------------------------------
# device-side helpers (torch only holds memory and names the stream)
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream, device):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def _logits(t, name="logits", seq_start=None):
    """rlo_logits view of a [rows, V] (or [B, T, V]) CUDA tensor.  seq_start:
    optional int64 CUDA tensor [B] (e.g. cu_seqlens[:-1]) for the packed /
    varlen layout, token (b, t) = row seq_start[b] + t."""
    torch = _torch()
    if t is None:
        return None
    if t.dtype == torch.float32:
        dt = _abi.DTYPE_F32
    elif t.dtype == torch.bfloat16:
        dt = _abi.DTYPE_BF16
    else:
        raise InputError(f"{name}: dtype must be float32 or bfloat16")
    if not t.is_cuda:
        raise InputError(f"{name}: must be a CUDA tensor")
    rows = t.reshape(-1, t.shape[-1]) if t.dim() != 2 else t
    if rows.stride(-1) != 1:
        raise InputError(f"{name}: vocab dimension must be contiguous")
    if t.dim() == 3 and t.stride(0) != t.shape[1] * t.stride(1):
        raise InputError(f"{name}: rows must be uniformly strided")
    stride = t.stride(-2) if t.dim() >= 2 and t.shape[-2] > 1 else t.shape[-1]  # a single row's stride is moot
    L = _abi.rlo_logits()
    L.data, L.dtype, L.V, L.row_stride = t.data_ptr(), dt, t.shape[-1], stride
    if seq_start is not None:
        _check_dev(seq_start, torch.int64, f"{name} seq_start")
        L.seq_start = seq_start.data_ptr()
    return L


def _batch(lengths, tokens, mask, T, seq_offset=0):
    b = _abi.rlo_batch()
    b.B, b.T, b.seq_offset = int(lengths.numel()), int(T), int(seq_offset)
    b.lengths = lengths.data_ptr()
    b.tokens = tokens.data_ptr() if tokens is not None else None
    b.mask = mask.data_ptr() if mask is not None else None
    return b


def _check_dev(t, dtype, name):
    torch = _torch()
    if t is None:
        return None
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise InputError(f"{name}: expected a contiguous CUDA tensor of {dtype}")
    return t


class Objective:
    """One handle per GPU per host thread (the reference's one PolicyWorkspace
    per worker, policy_workers.hpp:41)."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = C.c_void_p()
        check(_abi.lib().rlo_create(self.device, C.byref(h)))
        self._h = h
        self.rank, self.world = 0, 1

    # -- data-parallel group ------------------------------------------------
    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_abi.lib().rlo_comm_unique_id(buf))
        return buf.raw

    def init_comm(self, unique_id: bytes, rank: int, world: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(_abi.lib().rlo_comm_init(self._h, buf, rank, world))
        self.rank, self.world = rank, world

    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().rlo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self, stream=None) -> None:
        check(_abi.lib().rlo_sync(self._h, _stream(stream, self.device)))

    # -- the path -------------------------------------------------------------
    def forward_logprobs(self, logits, tokens, lengths, entropy=False, token_logit=False, seq_start=None,
                         stream=None):
        """forward_logprobs (policy.cpp:210-233): log-prob of every valid
        response position.  logits [B,T,V] or [B*T,V]; tokens [B,T] int32;
        lengths [B] int32.  Returns dict of float32 [B,T] tensors."""
        torch = _torch()
        B, T = tokens.shape
        _check_dev(tokens, torch.int32, "tokens")
        _check_dev(lengths, torch.int32, "lengths")
        out = {"logp": torch.empty(B, T, dtype=torch.float32, device=tokens.device)}
        if entropy:
            out["entropy"] = torch.empty_like(out["logp"])
        if token_logit:
            out["token_logit"] = torch.empty_like(out["logp"])
        check(_abi.lib().rlo_forward_logprobs(
            self._h, C.byref(_batch(lengths, tokens, None, T)), C.byref(_logits(logits, seq_start=seq_start)),
            _ptr(out["logp"]),
            _ptr(out.get("entropy")), _ptr(out.get("token_logit")), _stream(stream, self.device)))
        return out

    def compute_advantages(self, cfg: TrainConfig, lengths, T=None, mask=None, rewards=None, scalar_rewards=None,
                           values=None, returns=False, out=None, stream=None):
        """compute_advantages (policy.cpp:257-311) + GRPO / GAE.  rewards [B,T]
        (per token) or scalar_rewards [B] (on the last token); values [B,T]."""
        torch = _torch()
        _check_dev(lengths, torch.int32, "lengths")
        for t, n in ((rewards, "rewards"), (scalar_rewards, "scalar_rewards"), (values, "values")):
            _check_dev(t, torch.float32, n)
        _check_dev(mask, torch.uint8, "mask")
        B = int(lengths.numel())
        if T is None:
            src = rewards if rewards is not None else (values if values is not None else mask)
            if src is None:
                raise InputError("compute_advantages: T must be given with scalar rewards only")
            T = src.shape[-1]
        adv = out if out is not None else torch.empty(B, T, dtype=torch.float32, device=lengths.device)
        ret = torch.empty_like(adv) if returns else None
        check(_abi.lib().rlo_compute_advantages(
            self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, None, mask, T)), _ptr(rewards),
            _ptr(scalar_rewards), _ptr(values), _ptr(adv), _ptr(ret), _stream(stream, self.device)))
        return (adv, ret) if returns else adv

    def ppo_gradient(self, cfg: TrainConfig, tokens, lengths, actor_logits, advantages, mask=None, old_logits=None,
                     ref_logits=None, old_logprobs=None, ref_logprobs=None, seq_offset=0,
                     outputs=("logp", "dlogp"), seq_start=None, stream=None):
        """ppo_gradient loss part (policy.cpp:313-374), fused over the logits.
        Accumulates per-sequence sums until merge_gradients().  Returns the
        requested per-token outputs ([B,T] float32): logp, old_logp, ref_logp,
        entropy, dlogp, loss, lse."""
        torch = _torch()
        B, T = tokens.shape
        _check_dev(tokens, torch.int32, "tokens")
        _check_dev(lengths, torch.int32, "lengths")
        _check_dev(mask, torch.uint8, "mask")
        for t, n in ((advantages, "advantages"), (old_logprobs, "old_logprobs"), (ref_logprobs, "ref_logprobs")):
            _check_dev(t, torch.float32, n)
        res = {k: torch.empty(B, T, dtype=torch.float64 if k == "lse64" else torch.float32, device=tokens.device)
               for k in outputs}
        o = _abi.rlo_token_out()
        for k in ("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss", "lse", "lse64"):
            setattr(o, k, res[k].data_ptr() if k in res else None)
        L_old = _logits(old_logits, "old_logits", seq_start)
        L_ref = _logits(ref_logits, "ref_logits", seq_start)
        check(_abi.lib().rlo_ppo_gradient(
            self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, tokens, mask, T, seq_offset)),
            C.byref(_logits(actor_logits, "actor_logits", seq_start)), C.byref(L_old) if L_old else None,
            C.byref(L_ref) if L_ref else None, _ptr(old_logprobs), _ptr(ref_logprobs), _ptr(advantages),
            C.byref(o), _stream(stream, self.device)))
        return res

    def merge_gradients(self, cfg: TrainConfig, stream=None, with_partials=False):
        """merge_gradients (policy.cpp:421-450) across the accumulated
        micro-batches and (with a communicator) all ranks.  Synchronises."""
        st, part = _abi.rlo_stats(), _abi.rlo_partials()
        check(_abi.lib().rlo_merge_gradients(self._h, C.byref(cfg.to_c()), C.byref(st), C.byref(part),
                                             _stream(stream, self.device)))
        stats = UpdateStats.from_c(st)
        return (stats, np.array(part.v[:])) if with_partials else stats

    def merge_gradients_async(self, cfg: TrainConfig, out=None, stream=None):
        """merge_gradients with no host synchronisation (CUDA-graph capturable):
        the merged UpdateStats and the error status land in `out`, a device
        uint8 tensor of sizeof(rlo_step_result) bytes (allocated when None).
        Read it with step_result()."""
        torch = _torch()
        if out is None:
            out = torch.zeros(C.sizeof(_abi.rlo_step_result), dtype=torch.uint8, device=self.device)
        check(_abi.lib().rlo_merge_gradients_async(self._h, C.byref(cfg.to_c()), C.c_void_p(out.data_ptr()),
                                                   _stream(stream, self.device)))
        return out

    @staticmethod
    def step_result(buf) -> UpdateStats:
        """UpdateStats of a merge_gradients_async result (copies it to the host);
        raises what the synchronous merge_gradients would have raised."""
        raw = bytes(buf.cpu().numpy().tobytes())
        r = _abi.rlo_step_result.from_buffer_copy(raw)
        check(_abi.lib().rlo_step_result_check(C.byref(r)))
        return UpdateStats.from_c(r.stats)

    # -- next rows: backward epilogue, critic ----------------------------------
    def loss_weights(self, cfg: TrainConfig, lengths, stats: "UpdateStats", T, mask=None, stream=None):
        """d(L)/d(loss_t) per token under cfg.loss_agg with the merged counts."""
        torch = _torch()
        st = _abi.rlo_stats()
        for f in fields(UpdateStats):
            setattr(st, f.name, getattr(stats, f.name))
        w = torch.empty(int(lengths.numel()), T, dtype=torch.float32, device=lengths.device)
        check(_abi.lib().rlo_loss_weights(self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, None, mask, T)),
                                          C.byref(st), _ptr(w), _stream(stream, self.device)))
        return w

    def batch_counts(self, cfg: TrainConfig, lengths, T, mask=None, stream=None) -> "UpdateStats":
        """Global token / sequence / group counts of a batch before its vocab
        pass (the normalisers merge_gradients derives); feeds loss_weights
        ahead of ppo_gradient_fused.  Synchronises."""
        st = _abi.rlo_stats()
        check(_abi.lib().rlo_batch_counts(self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, None, mask, T)),
                                          C.byref(st), _stream(stream, self.device)))
        return UpdateStats.from_c(st)

    def ppo_gradient_fused(self, cfg: TrainConfig, tokens, lengths, actor_logits, advantages, weight, mask=None,
                           old_logits=None, ref_logits=None, old_logprobs=None, ref_logprobs=None, seq_offset=0,
                           grad=None, grad_dtype=None, outputs=("logp", "dlogp"), seq_start=None, stream=None):
        """ppo_gradient + the actor backward epilogue in one read of the actor
        logits (policy.cpp:355-379).  Accumulates like ppo_gradient; returns
        (per-token outputs dict, grad [B*T, V])."""
        torch = _torch()
        B, T = tokens.shape
        _check_dev(tokens, torch.int32, "tokens")
        _check_dev(lengths, torch.int32, "lengths")
        _check_dev(mask, torch.uint8, "mask")
        for t, n in ((advantages, "advantages"), (old_logprobs, "old_logprobs"), (ref_logprobs, "ref_logprobs"),
                     (weight, "weight")):
            _check_dev(t, torch.float32, n)
        if grad is None:
            grad = torch.empty(B * T, actor_logits.shape[-1], dtype=grad_dtype or actor_logits.dtype,
                               device=actor_logits.device)
        G = _logits(grad, "grad")
        res = {k: torch.empty(B, T, dtype=torch.float64 if k == "lse64" else torch.float32, device=tokens.device)
               for k in outputs}
        o = _abi.rlo_token_out()
        for k in ("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss", "lse", "lse64"):
            setattr(o, k, res[k].data_ptr() if k in res else None)
        L_old = _logits(old_logits, "old_logits", seq_start)
        L_ref = _logits(ref_logits, "ref_logits", seq_start)
        check(_abi.lib().rlo_ppo_gradient_fused(
            self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, tokens, mask, T, seq_offset)),
            C.byref(_logits(actor_logits, "actor_logits", seq_start)), C.byref(L_old) if L_old else None,
            C.byref(L_ref) if L_ref else None, _ptr(old_logprobs), _ptr(ref_logprobs), _ptr(advantages),
            _ptr(weight), C.c_void_p(grad.data_ptr()), G.dtype, G.row_stride, C.byref(o),
            _stream(stream, self.device)))
        return res, grad

    def logits_backward(self, tokens, lengths, logits, lse, dlogp, weight, grad=None, grad_dtype=None, seq_start=None,
                        stream=None):
        """Actor backward epilogue (policy.cpp:375-379): dL/dlogits rows
        w*dlogp*(onehot - softmax); returns the gradient tensor.  lse: the
        ppo_gradient "lse" (fp32) or "lse64" (fp64, exact at any logit offset)."""
        torch = _torch()
        B, T = tokens.shape
        if grad is None:
            grad = torch.empty(B * T, logits.shape[-1], dtype=grad_dtype or logits.dtype, device=logits.device)
        G = _logits(grad, "grad")
        fn = _abi.lib().rlo_logits_backward64 if lse.dtype == torch.float64 else _abi.lib().rlo_logits_backward
        check(fn(
            self._h, C.byref(_batch(lengths, tokens, None, T)), C.byref(_logits(logits, seq_start=seq_start)), _ptr(lse),
            _ptr(dlogp),
            _ptr(weight), C.c_void_p(grad.data_ptr()), G.dtype, G.row_stride, _stream(stream, self.device)))
        return grad

    def value_loss(self, lengths, values, returns, old_values=None, value_clip=0.0, mask=None, dvalue=True,
                   stream=None):
        """Critic value loss (value_gradient, policy.cpp:474-540); returns (stats dict, dvalue)."""
        torch = _torch()
        B, T = values.shape
        dv = torch.empty_like(values) if dvalue else None
        st = _abi.rlo_value_stats()
        check(_abi.lib().rlo_value_loss(self._h, C.byref(_batch(lengths, None, mask, T)), _ptr(values),
                                        _ptr(old_values), _ptr(returns), C.c_double(value_clip), _ptr(dv),
                                        C.byref(st), _stream(stream, self.device)))
        return {k: getattr(st, k) for k, _ in st._fields_}, dv

    def broadcast_params(self, buffer, bucket_bytes: int, root: int = 0, stream=None) -> None:
        """ModelUpdateGroup: bucketed NCCL broadcast of a device tensor from `root`
        (sync_params, policy_workers.cpp:234-260)."""
        check(_abi.lib().rlo_broadcast_params(self._h, C.c_void_p(buffer.data_ptr()),
                                              buffer.numel() * buffer.element_size(), bucket_bytes, root,
                                              _stream(stream, self.device)))

    def decode_sample(self, logits, temperature, seed, version, sample_keys, positions, stream=None):
        """decode_next (policy.cpp:143-169) per row: (tokens int32, untempered logp float32)."""
        torch = _torch()
        n = logits.numel() // logits.shape[-1]
        _check_dev(sample_keys, torch.int64, "sample_keys")
        _check_dev(positions, torch.int64, "positions")
        tok = torch.empty(n, dtype=torch.int32, device=logits.device)
        lp = torch.empty(n, dtype=torch.float32, device=logits.device)
        check(_abi.lib().rlo_decode_sample(self._h, C.byref(_logits(logits)), n, C.c_double(temperature),
                                           C.c_uint64(seed), C.c_uint64(version), _ptr(sample_keys), _ptr(positions),
                                           _ptr(tok), _ptr(lp), _stream(stream, self.device)))
        return tok, lp

    def rank_partials(self, cfg: TrainConfig, stream=None) -> np.ndarray:
        """This rank's GradAccum scalars (no cross-rank merge, no checks); resets."""
        part = _abi.rlo_partials()
        check(_abi.lib().rlo_rank_partials(self._h, C.byref(cfg.to_c()), C.byref(part),
                                           _stream(stream, self.device)))
        return np.array(part.v[:])

    def step(self, cfg: TrainConfig, tokens, lengths, actor_logits, mask=None, rewards=None, scalar_rewards=None,
             values=None, old_logits=None, ref_logits=None, old_logprobs=None, ref_logprobs=None, adv_out=None,
             stream=None) -> UpdateStats:
        """The whole path on device-resident inputs (rlo_objective_step)."""
        B, T = tokens.shape
        st = _abi.rlo_stats()
        L_old, L_ref = _logits(old_logits, "old_logits"), _logits(ref_logits, "ref_logits")
        check(_abi.lib().rlo_objective_step(
            self._h, C.byref(cfg.to_c()), C.byref(_batch(lengths, tokens, mask, T)), _ptr(rewards),
            _ptr(scalar_rewards), _ptr(values), C.byref(_logits(actor_logits, "actor_logits")),
            C.byref(L_old) if L_old else None, C.byref(L_ref) if L_ref else None, _ptr(old_logprobs),
            _ptr(ref_logprobs), _ptr(adv_out), None, C.byref(st), _stream(stream, self.device)))
        return UpdateStats.from_c(st)

    def step_host(self, cfg: TrainConfig, tokens: np.ndarray, lengths: np.ndarray, actor_logits, mask=None,
                  rewards=None, scalar_rewards=None, values=None, old_logits=None, ref_logits=None,
                  old_logprobs=None, ref_logprobs=None, adv_out=None, logp_out=None, stream=None) -> UpdateStats:
        """Reference-facing form: SampleBatch arrays in (pinned) host memory,
        copied in and results copied out inside the call."""
        B, T = tokens.shape
        st = _abi.rlo_stats()

        def hp(a):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):
                return C.c_void_p(a.data_ptr())
            return a.ctypes.data_as(C.c_void_p)

        L_old, L_ref = _logits(old_logits, "old_logits"), _logits(ref_logits, "ref_logits")
        check(_abi.lib().rlo_objective_step_host(
            self._h, C.byref(cfg.to_c()), B, T, hp(lengths), hp(tokens), hp(mask), hp(rewards), hp(scalar_rewards),
            hp(values), C.byref(_logits(actor_logits, "actor_logits")), C.byref(L_old) if L_old else None,
            C.byref(L_ref) if L_ref else None, hp(old_logprobs), hp(ref_logprobs), hp(adv_out), hp(logp_out),
            C.byref(st), _stream(stream, self.device)))
        return UpdateStats.from_c(st)


    def step_host_mb(self, cfg: TrainConfig, tokens: np.ndarray, lengths: np.ndarray, mb_seqs: int, logits_fn,
                     mask=None, rewards=None, scalar_rewards=None, values=None, old_logprobs=None,
                     ref_logprobs=None, adv_out=None, logp_out=None, stream=None) -> UpdateStats:
        """Micro-batched reference-facing step (rlo_objective_step_host_mb):
        host SampleBatch arrays for the whole batch, advantages over the whole
        batch, then ``logits_fn(i, seq_begin, n_seqs)`` -> (actor, old, ref)
        device tensors (old/ref may be None) names each micro-batch's logits
        (called on this thread, in order, before that micro-batch's pass)."""
        B, T = tokens.shape
        st = _abi.rlo_stats()
        keep = []
        err = []

        def hp(a):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):
                return C.c_void_p(a.data_ptr())
            return a.ctypes.data_as(C.c_void_p)

        def cb(_user, i, b0, nb, pa, po, pr):
            try:
                ts = logits_fn(int(i), int(b0), int(nb))
                for t, dst in zip(ts, (pa, po, pr)):
                    if t is not None:
                        L = _logits(t)
                        keep.append(t)
                        dst[0] = L
                return 0
            except Exception as e:  # surfaced after the call returns
                err.append(e)
                return _abi.RLO_ERR_INPUT

        fn = _abi.LOGITS_FN(cb)
        rc = _abi.lib().rlo_objective_step_host_mb(
            self._h, C.byref(cfg.to_c()), B, T, mb_seqs, hp(lengths), hp(tokens), hp(mask), hp(rewards),
            hp(scalar_rewards), hp(values), fn, None, hp(old_logprobs), hp(ref_logprobs), hp(adv_out), hp(logp_out),
            C.byref(st), _stream(stream, self.device))
        if err:
            raise err[0]
        check(rc)
        return UpdateStats.from_c(st)


def synth_logits(dst, seed: int, model: int, row_key_offset: int = 0, stream=None) -> None:
    """Fill a [rows, V] (row-strided) float32/bfloat16 CUDA tensor with the
    deterministic synthetic logits of include/rlo_synth.h."""
    L = _logits(dst, "dst")
    rows = dst.numel() // dst.shape[-1]
    check(_abi.lib().rlo_synth_logits(C.c_void_p(dst.data_ptr()), L.dtype, rows, L.V, L.row_stride, seed, model,
                                      row_key_offset, _stream(stream, dst.device)))


def synth_tokens(dst, V: int, seed: int, row_key_offset: int = 0, key_rows: int | None = None, stream=None) -> None:
    rows = dst.numel()
    check(_abi.lib().rlo_synth_tokens(C.c_void_p(dst.data_ptr()), rows, V, seed, row_key_offset,
                                      key_rows or rows, _stream(stream, dst.device)))


@dataclass
class Message:
    """worker.hpp:20-31: batch (tensors of the padded SampleBatch) + control plane."""

    batch: dict = field(default_factory=dict)
    tensors: dict = field(default_factory=dict)
    scalars: dict = field(default_factory=dict)
    fields: dict = field(default_factory=dict)


class PolicyWorker:
    """Worker plugin for the path's methods (policy_workers.cpp:46-64):
    ``forward_logprobs`` fills ``batch['ref_logprobs']`` (:93-100);
    ``compute_gradient`` returns the GradAccum scalars and ``tensors['grad']``
    (:111-121) -- 0-dim here, the model backward belongs to the trainer --
    plus ``tensors['dlogp']``; ``apply_update`` (:123-128, policy.cpp:452-460)
    advances the version (a zero learning rate is no update) and hands the
    step to ``on_update(learning_rate, grad_mean, version)``; ``get_version``.
    The batch carries the model's logits under ``batch['logits']``."""

    METHODS = ("forward_logprobs", "compute_gradient", "apply_update", "get_version")

    def __init__(self, device: int, train_config: TrainConfig, rank: int = 0, world_size: int = 1,
                 on_update=None):
        train_config.validate()
        self.rank, self.world_size, self.device_id = rank, world_size, f"cuda:{device}"
        self.train_config = train_config
        self.obj = Objective(device)
        self.version = 1
        self.on_update = on_update

    def call(self, method: str, msg: Message) -> Message:
        if method == "forward_logprobs":
            b = msg.batch
            lp = self.obj.forward_logprobs(b["logits"], b["response_tokens"], b["lengths"])["logp"]
            out = Message(batch=dict(b), fields={"version": str(self.version)})
            out.batch["ref_logprobs"] = lp
            return out
        if method == "compute_gradient":
            b = msg.batch
            res = self.obj.ppo_gradient(self.train_config, b["response_tokens"], b["lengths"], b["logits"],
                                        b["advantages"], mask=b.get("action_mask"),
                                        old_logprobs=b["response_logprobs"], ref_logprobs=b.get("ref_logprobs"),
                                        outputs=("dlogp",))
            p = self.obj.rank_partials(self.train_config)
            out = Message()
            out.tensors = {"grad": [], "dlogp": res["dlogp"]}
            out.scalars = {"loss_sum": p[0], "ratio_sum": p[1], "kl_sum": p[2], "clipped": p[4], "tokens": p[6]}
            return out
        if method == "apply_update":
            lr = float(msg.scalars["learning_rate"])
            grad_mean = msg.tensors.get("grad_mean", [])
            if lr != 0.0:
                self.version += 1
                if self.on_update is not None:
                    self.on_update(lr, grad_mean, self.version)
            return Message(fields={"version": str(self.version)})
        if method == "get_version":
            return Message(fields={"version": str(self.version)})
        raise DispatchError(f"policy worker: unimplemented method '{method}'")


def cluster_train_step(workers, shards, config: TrainConfig) -> UpdateStats:
    """cluster_train_step (policy_workers.cpp:208-232) over in-process workers:
    compute_gradient on each rank's shard, merge_gradients of the rank-ordered
    GradAccum scalars (policy.cpp:421-450), apply_update broadcast."""
    replies = [w.call("compute_gradient", Message(batch=s)) for w, s in zip(workers, shards)]
    parts = np.zeros((len(replies), _abi.NPARTIAL))
    for r, rep in enumerate(replies):
        parts[r, [0, 1, 2, 4, 6]] = [rep.scalars[k] for k in ("loss_sum", "ratio_sum", "kl_sum", "clipped", "tokens")]
    stats = merge_partials(parts, config)
    for w in workers:
        w.call("apply_update", Message(tensors={"grad_mean": []}, scalars={"learning_rate": config.learning_rate}))
    return stats


def sample_key(sample_id: str) -> int:
    """rng::hash_str (rng.hpp:34-41): the per-sample key decode_next draws with."""
    return int(_abi.lib().rlo_sample_key(sample_id.encode()))


def batch_from_jsonl(text) -> dict:
    """SampleBatch::from_jsonl (sample.cpp:150-158) + validate, into padded numpy arrays
    (keys of rlo_host_batch; absent arrays are None)."""
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    hb = C.POINTER(_abi.rlo_host_batch)()
    check(_abi.lib().rlo_batch_from_jsonl(data, len(data), C.byref(hb)))
    try:
        b = hb.contents
        B, T = b.B, b.T
        out = {"B": B, "T": T, "first_missing_reward": b.first_missing_reward}

        def arr(ptr, n, shape):
            return None if not ptr else np.ctypeslib.as_array(ptr, shape=(n,)).copy().reshape(shape)

        out["lengths"] = arr(b.lengths, B, (B,))
        out["tokens"] = arr(b.tokens, B * T, (B, T))
        out["mask"] = arr(b.mask, B * T, (B, T))
        for k in ("rewards", "response_logprobs", "ref_logprobs", "advantages"):
            out[k] = arr(getattr(b, k), B * T, (B, T))
        out["scalar_rewards"] = arr(b.scalar_rewards, B, (B,))
        out["sample_keys"] = arr(b.sample_keys, B, (B,))
        out["group_index"] = arr(b.group_index, B, (B,))
        return out
    finally:
        _abi.lib().rlo_host_batch_free(hb)


def bucket_plan(total: int, bucket: int) -> list[int]:
    """bucket_plan (policy.cpp:542-548)."""
    n = C.c_int64(0)
    _abi.lib().rlo_bucket_plan(total, bucket, None, C.byref(n))  # sizing call
    out = (C.c_uint64 * max(1, n.value))()
    check(_abi.lib().rlo_bucket_plan(total, bucket, out, C.byref(n)))
    return list(out[:n.value])
