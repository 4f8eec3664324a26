"""ctypes bindings of the CPU oracle (oracle/liboracle.so) and of the
reference's own code (oracle/_ref/librollmini_ref.so).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs import this package,
and only as the checker or the timed CPU baseline.  The product
(``paper_2506_06122_b200``) never imports it.

Every wrapper returns numpy arrays in the padded [B, T] layout of
``include/rlo.h``.  Non-OK status codes raise the same exception classes the
product raises (``paper_2506_06122_b200.errors``-compatible names are
re-declared here so the oracle has no dependency on the product).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librollmini_ref.so")

RLO_OK, RLO_ERR_INPUT, RLO_ERR_CONFIG, RLO_ERR_TRAINING = 0, 1, 2, 3
F32, BF16 = 0, 1
REINFORCE, GRPO, GAE = 0, 1, 2
K1, K2, K3 = 0, 1, 2
TOKEN_MEAN, SEQ_MEAN_TOKEN_MEAN, SEQ_MEAN_TOKEN_SUM, GROUP_MEAN = 0, 1, 2, 3
NPARTIAL = 16


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class TrainConfig(C.Structure):
    """Mirror of ``rlo_train_config`` (include/rlo.h)."""

    _fields_ = [
        ("clip_eps", C.c_double), ("kl_coef", C.c_double), ("learning_rate", C.c_double),
        ("advantage_clip", C.c_double), ("reward_clip", C.c_double), ("gamma", C.c_double),
        ("whiten_advantages", C.c_int32), ("adv_estimator", C.c_int32), ("lambd", C.c_double),
        ("kl_estimator", C.c_int32), ("dual_clip_c", C.c_double), ("loss_agg", C.c_int32),
        ("group_size", C.c_int32), ("grpo_std_ddof", C.c_int32), ("grpo_eps", C.c_double),
    ]

    def __init__(self, **kw):
        super().__init__()
        d = dict(clip_eps=0.2, kl_coef=0.0, learning_rate=0.05, advantage_clip=10.0, reward_clip=20.0,
                 gamma=1.0, whiten_advantages=0, adv_estimator=REINFORCE, lambd=0.95, kl_estimator=K1,
                 dual_clip_c=0.0, loss_agg=TOKEN_MEAN, group_size=1, grpo_std_ddof=0, grpo_eps=1e-6)
        d.update(kw)
        for k, v in d.items():
            setattr(self, k, int(v) if isinstance(v, bool) else v)


class Partials(C.Structure):
    _fields_ = [("v", C.c_double * NPARTIAL)]


class Stats(C.Structure):
    _fields_ = [
        ("loss", C.c_double), ("mean_ratio", C.c_double), ("clip_fraction", C.c_double),
        ("mean_kl", C.c_double), ("tokens", C.c_uint64), ("mean_entropy", C.c_double),
        ("dual_clip_fraction", C.c_double), ("seqs", C.c_uint64), ("groups", C.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_ref = None


def build(with_ref: bool | None = None) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/core/src")
    if with_ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(with_ref=False)
        _lib = C.CDLL(ORACLE_SO)
        _lib.orc_bench_objective.restype = C.c_double
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        _ref = C.CDLL(REF_SO)
        _ref.ref_bench_objective.restype = C.c_double
    return _ref


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _u8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint8)


def _check(code, err):
    if code != RLO_OK:
        raise OracleError(code, err.value.decode())


# ---- oracle restatement -----------------------------------------------------

def logsoftmax_row(z):
    z = _f64(z)
    lse, ent = C.c_double(), C.c_double()
    lib().orc_logsoftmax_row(_p(z), C.c_int32(z.size), C.byref(lse), C.byref(ent))
    return lse.value, ent.value


def forward_logprobs(logits, dtype, V, row_stride, B, T, lengths, tokens):
    """logits: host array (float32 or uint16 bf16 bits), flat rows."""
    logits = np.ascontiguousarray(logits)
    lengths, tokens = _i32(lengths), _i32(tokens)
    lp, ent, tl = (np.zeros(B * T) for _ in range(3))
    err = C.create_string_buffer(512)
    code = lib().orc_forward_logprobs(_p(logits), C.c_int32(dtype), C.c_int32(V), C.c_int64(row_stride),
                                      C.c_int32(B), C.c_int32(T), _p(lengths), _p(tokens),
                                      _p(lp), _p(ent), _p(tl), err, C.c_int32(512))
    _check(code, err)
    return lp, ent, tl


def compute_advantages(cfg, B, T, lengths, mask=None, rewards_tok=None, rewards_seq=None, values=None):
    lengths, mask = _i32(lengths), _u8(mask)
    rewards_tok, rewards_seq, values = _f64(rewards_tok), _f64(rewards_seq), _f64(values)
    adv, ret = np.zeros(B * T), np.zeros(B * T)
    err = C.create_string_buffer(512)
    code = lib().orc_compute_advantages(C.byref(cfg), C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask),
                                        _p(rewards_tok), _p(rewards_seq), _p(values), _p(adv), _p(ret),
                                        err, C.c_int32(512))
    _check(code, err)
    return adv, ret


def ppo_loss(cfg, B, T, lengths, mask, lp, old_lp, ref_lp, adv, entropy=None):
    lengths, mask = _i32(lengths), _u8(mask)
    lp, old_lp, ref_lp, adv, entropy = map(_f64, (lp, old_lp, ref_lp, adv, entropy))
    loss_tok, dlogp = np.zeros(B * T), np.zeros(B * T)
    part = Partials()
    err = C.create_string_buffer(512)
    code = lib().orc_ppo_loss(C.byref(cfg), C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask), _p(lp),
                              _p(old_lp), _p(ref_lp), _p(adv), _p(entropy), _p(loss_tok), _p(dlogp),
                              C.byref(part), err, C.c_int32(512))
    _check(code, err)
    return loss_tok, dlogp, np.array(part.v[:])


def merge(parts, cfg):
    parts = np.ascontiguousarray(np.atleast_2d(parts), dtype=np.float64)
    arr = (Partials * len(parts))()
    for i, p in enumerate(parts):
        arr[i].v[:] = list(p)
    st = Stats()
    err = C.create_string_buffer(512)
    code = lib().orc_merge(arr, C.c_int32(len(parts)), C.byref(cfg), C.byref(st), err, C.c_int32(512))
    _check(code, err)
    return st.as_dict()


def split_sizes(n, parts):
    out = np.zeros(parts, dtype=np.int64)
    lib().orc_split_sizes(C.c_int64(n), C.c_int32(parts), _p(out))
    return out


def synth_row(dtype, V, seed, model, row_key):
    out = np.zeros(V)
    lib().orc_synth_row(_p(out), C.c_int32(dtype), C.c_int32(V), C.c_uint64(seed), C.c_int32(model),
                        C.c_uint64(row_key))
    return out


def synth_row_raw(dtype, V, seed, model, row_key):
    out = np.zeros(V, dtype=np.float32 if dtype == F32 else np.uint16)
    lib().orc_synth_row_raw(_p(out), C.c_int32(dtype), C.c_int32(V), C.c_uint64(seed), C.c_int32(model),
                            C.c_uint64(row_key))
    return out


def synth_token(seed, row_key, V):
    return int(lib().orc_synth_token(C.c_uint64(seed), C.c_uint64(row_key), C.c_int32(V)))


def bench_objective(threads, cfg, dtype, V, B, T, key_rows, seed, use_ref=False):
    """Times the CPU path on a bounded sample; returns (seconds, loss checksum)."""
    chk = C.c_double()
    fn = ref().ref_bench_objective if use_ref else lib().orc_bench_objective
    secs = fn(C.c_int32(threads), C.byref(cfg), C.c_int32(dtype), C.c_int32(V), C.c_int32(B), C.c_int32(T),
              C.c_int32(key_rows), C.c_uint64(seed), C.byref(chk))
    return float(secs), chk.value


# ---- the reference's own code (oracle/_ref) ---------------------------------

def ref_logsoftmax_rows(rows, toks, full=False):
    rows = _f64(np.atleast_2d(rows))
    n, V = rows.shape
    toks = _i32(toks)
    lp = np.zeros(n)
    fullout = np.zeros((n, V)) if full else None
    err = C.create_string_buffer(512)
    code = ref().ref_logsoftmax_rows(_p(rows), C.c_int32(n), C.c_int32(V), _p(toks), _p(lp), _p(fullout), err,
                                     C.c_int32(512))
    _check(code, err)
    return (lp, fullout) if full else lp


def ref_forward_logprobs_b2(row, B, T, lengths, tokens):
    row, lengths, tokens = _f64(row), _i32(lengths), _i32(tokens)
    out = np.zeros(B * T)
    err = C.create_string_buffer(512)
    code = ref().ref_forward_logprobs_b2(_p(row), C.c_int32(row.size), C.c_int32(B), C.c_int32(T), _p(lengths),
                                         _p(tokens), _p(out), err, C.c_int32(512))
    _check(code, err)
    return out


def ref_compute_advantages(cfg, B, T, lengths, mask=None, rewards_tok=None, rewards_seq=None):
    lengths, mask, rewards_tok, rewards_seq = _i32(lengths), _u8(mask), _f64(rewards_tok), _f64(rewards_seq)
    out = np.zeros(B * T)
    err = C.create_string_buffer(512)
    code = ref().ref_compute_advantages(C.byref(cfg), C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask),
                                        _p(rewards_tok), _p(rewards_seq), _p(out), err, C.c_int32(512))
    _check(code, err)
    return out


def ref_ppo_stats_b2(row, B, T, lengths, tokens, mask, old_lp, ref_lp, adv, cfg, world=1):
    row, lengths, tokens, mask = _f64(row), _i32(lengths), _i32(tokens), _u8(mask)
    old_lp, ref_lp, adv = _f64(old_lp), _f64(ref_lp), _f64(adv)
    out = np.zeros(5)
    err = C.create_string_buffer(512)
    code = ref().ref_ppo_stats_b2(_p(row), C.c_int32(row.size), C.c_int32(B), C.c_int32(T), _p(lengths),
                                  _p(tokens), _p(mask), _p(old_lp), _p(ref_lp), _p(adv), C.byref(cfg),
                                  C.c_int32(world), _p(out), err, C.c_int32(512))
    _check(code, err)
    return dict(zip(["loss", "mean_ratio", "clip_fraction", "mean_kl", "tokens"], out.tolist()))


def ref_merge_scalars(parts5):
    parts5 = _f64(np.atleast_2d(parts5))
    out = np.zeros(5)
    err = C.create_string_buffer(512)
    code = ref().ref_merge_scalars(_p(parts5), C.c_int32(parts5.shape[0]), _p(out), err, C.c_int32(512))
    _check(code, err)
    return dict(zip(["loss", "mean_ratio", "clip_fraction", "mean_kl", "tokens"], out.tolist()))


def ref_train_config_validate(cfg):
    err = C.create_string_buffer(512)
    code = ref().ref_train_config_validate(C.byref(cfg), err, C.c_int32(512))
    return code, err.value.decode()


def ref_split_sizes(n, parts):
    out = np.zeros(parts, dtype=np.int64)
    ref().ref_split_sizes(C.c_int64(n), C.c_int32(parts), _p(out))
    return out


# ---- aggregation weights, actor backward, value loss ---------------------------

def loss_weights(cfg, B, T, lengths, mask=None):
    lengths, mask = _i32(lengths), _u8(mask)
    out = np.zeros(B * T)
    lib().orc_loss_weights(C.byref(cfg), C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask), _p(out))
    return out


def logits_backward_row(z, tok, scale):
    z = _f64(z)
    out = np.zeros(z.size)
    lib().orc_logits_backward_row(_p(z), C.c_int32(z.size), C.c_int32(tok), C.c_double(scale), _p(out))
    return out


def value_loss(B, T, lengths, mask, values, old_values, returns, value_clip=0.0):
    lengths, mask = _i32(lengths), _u8(mask)
    values, old_values, returns = _f64(values), _f64(old_values), _f64(returns)
    dv, out4 = np.zeros(B * T), np.zeros(4)
    lib().orc_value_loss(C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask), _p(values), _p(old_values),
                         _p(returns), C.c_double(value_clip), _p(dv), _p(out4))
    return dv, dict(zip(["loss_sum", "tokens", "clipped", "value_sum"], out4.tolist()))


def ref_ppo_grad_b2(row, B, T, lengths, tokens, mask, old_lp, ref_lp, adv, cfg, world=1):
    row, lengths, tokens, mask = _f64(row), _i32(lengths), _i32(tokens), _u8(mask)
    old_lp, ref_lp, adv = _f64(old_lp), _f64(ref_lp), _f64(adv)
    out = np.zeros(row.size)
    err = C.create_string_buffer(512)
    code = ref().ref_ppo_grad_b2(_p(row), C.c_int32(row.size), C.c_int32(B), C.c_int32(T), _p(lengths),
                                 _p(tokens), _p(mask), _p(old_lp), _p(ref_lp), _p(adv), C.byref(cfg),
                                 C.c_int32(world), _p(out), err, C.c_int32(512))
    _check(code, err)
    return out


def ref_value_loss_b2(vb, B, T, lengths, mask, targets):
    lengths, mask, targets = _i32(lengths), _u8(mask), _f64(targets)
    out = np.zeros(3)
    err = C.create_string_buffer(512)
    code = ref().ref_value_loss_b2(C.c_double(vb), C.c_int32(B), C.c_int32(T), _p(lengths), _p(mask),
                                   _p(targets), _p(out), err, C.c_int32(512))
    _check(code, err)
    return dict(zip(["loss_sum", "tokens", "grad_vb"], out.tolist()))


# ---- decode_next (sampling-time log-probs) ------------------------------------

def decode_next(z, temperature, seed, version, sample_key, position):
    z = _f64(z)
    lp = C.c_double()
    tok = lib().orc_decode_next(_p(z), C.c_int32(z.size), C.c_double(temperature), C.c_uint64(seed),
                                C.c_uint64(version), C.c_uint64(sample_key), C.c_uint64(position), C.byref(lp))
    return int(tok), lp.value


def hash_str(s):
    lib().orc_hash_str.restype = C.c_uint64
    return int(lib().orc_hash_str(s.encode()))


def ref_decode_b2(row, temperature, seed, version, sample_key, position):
    row = _f64(row)
    tok, lp = C.c_int32(), C.c_double()
    err = C.create_string_buffer(512)
    code = ref().ref_decode_b2(_p(row), C.c_int32(row.size), C.c_double(temperature), C.c_uint64(seed),
                               C.c_uint64(version), C.c_uint64(sample_key), C.c_uint64(position), C.byref(tok),
                               C.byref(lp), err, C.c_int32(512))
    _check(code, err)
    return tok.value, lp.value


def ref_hash_str(s):
    ref().ref_hash_str.restype = C.c_uint64
    return int(ref().ref_hash_str(s.encode()))


# ---- wire format / bucket plan ------------------------------------------------

def ref_batch_jsonl(seed, n):
    """SampleBatch::to_jsonl (sample.cpp:144-148) of a random batch (reference code)."""
    size = ref().ref_batch_jsonl(C.c_uint64(seed), C.c_int32(n), None, C.c_int64(0))
    ref().ref_batch_jsonl.restype = C.c_int64
    size = ref().ref_batch_jsonl(C.c_uint64(seed), C.c_int32(n), None, C.c_int64(0))
    buf = C.create_string_buffer(int(size) + 1)
    ref().ref_batch_jsonl(C.c_uint64(seed), C.c_int32(n), buf, C.c_int64(size))
    return buf.raw[:size].decode("utf-8")


def ref_bucket_plan(total, bucket):
    out = np.zeros(max(1, -(-total // bucket)) + 1, dtype=np.uint64)
    n = C.c_int64()
    ref().ref_bucket_plan(C.c_uint64(total), C.c_uint64(bucket), _p(out), C.byref(n))
    return out[:n.value].tolist()


def ref_parse_validate_jsonl(text):
    """(code, message) of SampleBatch::from_jsonl(text).validate() in the reference."""
    err = C.create_string_buffer(512)
    code = ref().ref_parse_validate_jsonl(text.encode("utf-8"), err, C.c_int32(512))
    return int(code), err.value.decode()
