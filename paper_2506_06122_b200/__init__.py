"""B200-native RL-objective hot path of ROLL (arXiv 2506.06122).

The product is ``lib/librlo.so`` (C ABI in ``include/rlo.h``, sm_100a
kernels in ``csrc/``).  This package mirrors the reference's host interface
(``include/rollmini/policy.hpp``, ``worker.hpp``) on top of that ABI.
"""
from ._abi import LIB_PATH, declared_symbols  # noqa: F401
from .errors import (CollectError, ConfigError, CudaError, DispatchError, Error, InputError,  # noqa: F401
                     TrainingError)
from .policy import (Message, batch_from_jsonl, bucket_plan, cluster_train_step, Objective, PolicyWorker, TrainConfig, UpdateStats, launch_count,  # noqa: F401
                     merge_partials, sample_key, shard_plan, split_sizes, synth_logits, synth_tokens,
                     whiten_combine)

__all__ = [
    "Objective", "PolicyWorker", "cluster_train_step", "Message", "TrainConfig", "UpdateStats", "split_sizes", "shard_plan",
    "merge_partials", "whiten_combine", "sample_key", "batch_from_jsonl", "bucket_plan", "launch_count", "synth_logits", "synth_tokens", "Error", "ConfigError", "InputError",
    "TrainingError", "DispatchError", "CollectError", "CudaError",
]
