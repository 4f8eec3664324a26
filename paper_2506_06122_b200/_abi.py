"""ctypes view of the C ABI (include/rlo.h) exported by lib/librlo.so.

The library is the product: this module only loads it and declares the
structures.  There is no fallback — if the CUDA library is missing the import
of any compute entry point fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# RLO_LIB overrides the in-tree library (A/B builds of the same sources in kernel experiments).
LIB_PATH = os.environ.get("RLO_LIB") or os.path.join(HERE, "lib", "librlo.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rlo.h")
ABI_VERSION = 5  # include/rlo.h RLO_ABI_VERSION: the struct layouts below

RLO_OK, RLO_ERR_INPUT, RLO_ERR_CONFIG, RLO_ERR_TRAINING, RLO_ERR_CUDA, RLO_ERR_NCCL, RLO_ERR_DISPATCH = range(7)
DTYPE_F32, DTYPE_BF16 = 0, 1
ADV_REINFORCE, ADV_GRPO, ADV_GAE = 0, 1, 2
KL_K1, KL_K2, KL_K3 = 0, 1, 2
AGG_TOKEN_MEAN, AGG_SEQ_MEAN_TOKEN_MEAN, AGG_SEQ_MEAN_TOKEN_SUM, AGG_GROUP_MEAN = 0, 1, 2, 3
NPARTIAL = 16


class rlo_train_config(C.Structure):
    _fields_ = [
        ("clip_eps", C.c_double), ("kl_coef", C.c_double), ("learning_rate", C.c_double),
        ("advantage_clip", C.c_double), ("reward_clip", C.c_double), ("gamma", C.c_double),
        ("whiten_advantages", C.c_int32), ("adv_estimator", C.c_int32), ("lambd", C.c_double),
        ("kl_estimator", C.c_int32), ("dual_clip_c", C.c_double), ("loss_agg", C.c_int32),
        ("group_size", C.c_int32), ("grpo_std_ddof", C.c_int32), ("grpo_eps", C.c_double),
    ]


class rlo_batch(C.Structure):
    _fields_ = [("B", C.c_int32), ("T", C.c_int32), ("seq_offset", C.c_int32), ("reserved", C.c_int32),
                ("lengths", C.c_void_p), ("tokens", C.c_void_p), ("mask", C.c_void_p)]


class rlo_logits(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("V", C.c_int32), ("row_stride", C.c_int64),
                ("seq_start", C.c_void_p)]


class rlo_token_out(C.Structure):
    _fields_ = [("logp", C.c_void_p), ("old_logp", C.c_void_p), ("ref_logp", C.c_void_p),
                ("entropy", C.c_void_p), ("dlogp", C.c_void_p), ("loss", C.c_void_p), ("lse", C.c_void_p),
                ("lse64", C.c_void_p)]


class rlo_stats(C.Structure):
    _fields_ = [
        ("loss", C.c_double), ("mean_ratio", C.c_double), ("clip_fraction", C.c_double),
        ("mean_kl", C.c_double), ("tokens", C.c_uint64), ("mean_entropy", C.c_double),
        ("dual_clip_fraction", C.c_double), ("seqs", C.c_uint64), ("groups", C.c_uint64),
    ]


class rlo_step_result(C.Structure):
    _fields_ = [("stats", rlo_stats), ("status", C.c_int32), ("reason", C.c_int32), ("dev_error", C.c_int32),
                ("dev_error_value", C.c_int32)]


class rlo_value_stats(C.Structure):
    _fields_ = [("loss", C.c_double), ("clip_fraction", C.c_double), ("mean_value", C.c_double),
                ("tokens", C.c_uint64)]


class rlo_host_batch(C.Structure):
    _fields_ = [("B", C.c_int32), ("T", C.c_int32), ("first_missing_reward", C.c_int32), ("reserved", C.c_int32),
                ("lengths", C.POINTER(C.c_int32)), ("tokens", C.POINTER(C.c_int32)), ("mask", C.POINTER(C.c_uint8)),
                ("rewards", C.POINTER(C.c_float)), ("scalar_rewards", C.POINTER(C.c_float)),
                ("response_logprobs", C.POINTER(C.c_float)), ("ref_logprobs", C.POINTER(C.c_float)),
                ("advantages", C.POINTER(C.c_float)), ("sample_keys", C.POINTER(C.c_uint64)),
                ("group_index", C.POINTER(C.c_int32))]


class rlo_partials(C.Structure):
    _fields_ = [("v", C.c_double * NPARTIAL)]


_lib = None


def declared_symbols() -> list[str]:
    """Every function include/rlo.h declares (used by the export test)."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"\btypedef\b[^;]*;", "", text)  # function-pointer types are not exports
    return sorted(set(re.findall(r"\b(rlo_[a-z0-9_]+)\s*\(", text)))


# rlo_logits_fn (include/rlo.h): the per-micro-batch logits callback of
# rlo_objective_step_host_mb.
LOGITS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(rlo_logits),
                        C.POINTER(rlo_logits), C.POINTER(rlo_logits))


def lib() -> C.CDLL:
    """Load librlo.so (built in-tree by __graft_entry__.build()); no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the sm_100a CUDA library must be built "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    P = C.POINTER
    sig = {
        "rlo_abi_version": ([], C.c_int),
        "rlo_last_error": ([], C.c_char_p),
        "rlo_launch_count": ([], u64),
        "rlo_train_config_default": ([P(rlo_train_config)], None),
        "rlo_train_config_validate": ([P(rlo_train_config)], C.c_int),
        "rlo_split_sizes": ([i64, i32, P(i64)], C.c_int),
        "rlo_shard_plan": ([i32, i32, i32, i32, P(i32), P(i32)], C.c_int),
        "rlo_merge_partials": ([P(rlo_partials), i32, P(rlo_train_config), P(rlo_stats)], C.c_int),
        "rlo_whiten_combine": ([vp, i32, P(C.c_double), P(C.c_double)], C.c_int32),
        "rlo_create": ([i32, P(vp)], C.c_int),
        "rlo_destroy": ([vp], C.c_int),
        "rlo_comm_unique_id": ([vp], C.c_int),
        "rlo_comm_init": ([vp, vp, i32, i32], C.c_int),
        "rlo_forward_logprobs": ([vp, P(rlo_batch), P(rlo_logits), vp, vp, vp, vp], C.c_int),
        "rlo_compute_advantages": ([vp, P(rlo_train_config), P(rlo_batch), vp, vp, vp, vp, vp, vp], C.c_int),
        "rlo_ppo_gradient": ([vp, P(rlo_train_config), P(rlo_batch), P(rlo_logits), P(rlo_logits),
                              P(rlo_logits), vp, vp, vp, P(rlo_token_out), vp], C.c_int),
        "rlo_merge_gradients": ([vp, P(rlo_train_config), P(rlo_stats), P(rlo_partials), vp], C.c_int),
        "rlo_rank_partials": ([vp, P(rlo_train_config), P(rlo_partials), vp], C.c_int),
        "rlo_merge_gradients_async": ([vp, P(rlo_train_config), vp, vp], C.c_int),
        "rlo_step_result_check": ([P(rlo_step_result)], C.c_int),
        "rlo_objective_step": ([vp, P(rlo_train_config), P(rlo_batch), vp, vp, vp, P(rlo_logits), P(rlo_logits),
                                P(rlo_logits), vp, vp, vp, P(rlo_token_out), P(rlo_stats), vp], C.c_int),
        "rlo_objective_step_host": ([vp, P(rlo_train_config), i32, i32, vp, vp, vp, vp, vp, vp, P(rlo_logits),
                                     P(rlo_logits), P(rlo_logits), vp, vp, vp, vp, P(rlo_stats), vp], C.c_int),
        "rlo_objective_step_host_mb": ([vp, P(rlo_train_config), i32, i32, i32, vp, vp, vp, vp, vp, vp,
                                        LOGITS_FN, vp, vp, vp, vp, vp, P(rlo_stats), vp], C.c_int),
        "rlo_sync": ([vp, vp], C.c_int),
        "rlo_loss_weights": ([vp, P(rlo_train_config), P(rlo_batch), P(rlo_stats), vp, vp], C.c_int),
        "rlo_logits_backward": ([vp, P(rlo_batch), P(rlo_logits), vp, vp, vp, vp, i32, i64, vp], C.c_int),
        "rlo_logits_backward64": ([vp, P(rlo_batch), P(rlo_logits), vp, vp, vp, vp, i32, i64, vp], C.c_int),
        "rlo_batch_counts": ([vp, P(rlo_train_config), P(rlo_batch), P(rlo_stats), vp], C.c_int),
        "rlo_ppo_gradient_fused": ([vp, P(rlo_train_config), P(rlo_batch), P(rlo_logits), P(rlo_logits),
                                    P(rlo_logits), vp, vp, vp, vp, vp, i32, i64, P(rlo_token_out), vp], C.c_int),
        "rlo_value_loss": ([vp, P(rlo_batch), vp, vp, vp, C.c_double, vp, P(rlo_value_stats), vp], C.c_int),
        "rlo_decode_sample": ([vp, P(rlo_logits), i32, C.c_double, u64, u64, vp, vp, vp, vp, vp], C.c_int),
        "rlo_sample_key": ([C.c_char_p], u64),
        "rlo_batch_from_jsonl": ([C.c_char_p, C.c_size_t, P(P(rlo_host_batch))], C.c_int),
        "rlo_host_batch_free": ([P(rlo_host_batch)], None),
        "rlo_bucket_plan": ([u64, u64, P(u64), P(i64)], C.c_int),
        "rlo_broadcast_params": ([vp, vp, u64, u64, i32, vp], C.c_int),
        "rlo_synth_logits": ([vp, i32, i64, i32, i64, u64, i32, i64, vp], C.c_int),
        "rlo_synth_tokens": ([vp, i64, i32, u64, i64, i64, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name, None)
        if fn is None and os.environ.get("RLO_LIB"):
            continue  # an older A/B build (RLO_LIB) may predate an entry point
        if fn is None:
            raise ImportError(f"{LIB_PATH} does not export {name}: rebuild the library")
        fn.argtypes = args
        fn.restype = res
    if L.rlo_abi_version() != ABI_VERSION and not os.environ.get("RLO_LIB"):
        raise ImportError(f"{LIB_PATH} has ABI version {L.rlo_abi_version()}, this binding expects {ABI_VERSION}: "
                          "rebuild the library")
    _lib = L
    return L
