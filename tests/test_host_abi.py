"""CPU tests of the C-ABI library's host side: it loads, exports every symbol
include/rlo.h declares, and its host logic (config validation, sharding,
rank-ordered merge) matches the reference (golden fixtures) and the oracle.
No compute calls (no GPU here)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2506_06122_b200 as rlo
from paper_2506_06122_b200 import _abi

G = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    declared = _abi.declared_symbols()
    assert len(declared) >= 21
    for s in declared:
        assert hasattr(L, s), s
    assert L.rlo_abi_version() == _abi.ABI_VERSION  # include/rlo.h RLO_ABI_VERSION


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_abi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    for arch in ("sm_80", "sm_90", "sm_90a"):
        assert f".{arch}." not in out


def test_config_defaults_are_reference_defaults():
    c = _abi.rlo_train_config()
    _abi.lib().rlo_train_config_default(C.byref(c))
    # policy.hpp:58-64
    assert (c.clip_eps, c.kl_coef, c.learning_rate, c.advantage_clip, c.reward_clip, c.gamma,
            c.whiten_advantages) == (0.2, 0.0, 0.05, 10.0, 20.0, 1.0, 0)
    d = rlo.TrainConfig()
    assert (d.clip_eps, d.kl_coef, d.learning_rate, d.advantage_clip, d.reward_clip, d.gamma) == \
        (0.2, 0.0, 0.05, 10.0, 20.0, 1.0)


def test_config_validation_messages_match_reference():
    for case in golden("misc.json")["train_config_validate"]:
        cfg = rlo.TrainConfig(**case["cfg"])
        if case["code"] == 0:
            cfg.validate()
        else:
            with pytest.raises(rlo.ConfigError) as e:
                cfg.validate()
            assert str(e.value) == case["msg"]


@pytest.mark.parametrize("kw,frag", [
    (dict(adv_estimator=7), "adv_estimator"), (dict(lambd=1.5), "lambda"), (dict(kl_estimator=5), "kl_estimator"),
    (dict(dual_clip_c=0.5), "dual_clip_c"), (dict(loss_agg=9), "loss_agg"), (dict(group_size=0), "group_size"),
    (dict(grpo_std_ddof=2), "grpo_std_ddof"), (dict(grpo_eps=-1.0), "grpo_eps")])
def test_extension_validation(kw, frag):
    with pytest.raises(rlo.ConfigError) as e:
        rlo.TrainConfig(**kw).validate()
    assert frag in str(e.value)


def test_split_sizes_match_reference():
    for c in golden("misc.json")["split_sizes"]:
        assert rlo.split_sizes(c["n"], c["parts"]) == c["sizes"]
    with pytest.raises(rlo.ConfigError):
        rlo.split_sizes(4, 0)


def test_shard_plan_is_group_aligned_and_covers_batch():
    for B, G, world in [(512, 8, 1), (512, 8, 2), (512, 8, 4), (8192, 8, 8), (96, 16, 4), (40, 8, 3), (7, 1, 4)]:
        spans = [rlo.shard_plan(B, G, world, r) for r in range(world)]
        pos = 0
        for b, n in spans:
            assert b == pos and b % G == 0 and n % G == 0
            pos += n
        assert pos == B
        sizes = [n for _, n in spans]
        assert sizes == sorted(sizes, reverse=True) and max(sizes) - min(sizes) <= G
    with pytest.raises(rlo.InputError):
        rlo.shard_plan(10, 4, 2, 0)


def test_merge_partials_matches_oracle_and_reference():
    rng = np.random.default_rng(1)
    for agg in range(4):
        parts = np.zeros((3, 16))
        parts[:, [0, 1, 2, 3, 7, 9]] = rng.standard_normal((3, 6))
        parts[:, 4] = rng.integers(0, 5, 3)
        parts[:, 5] = rng.integers(0, 3, 3)
        parts[:, 6] = rng.integers(5, 50, 3)
        parts[:, 8] = rng.integers(1, 5, 3)
        parts[:, 10] = rng.integers(1, 3, 3)
        st = rlo.merge_partials(parts, rlo.TrainConfig(loss_agg=agg))
        want = O.merge(parts, O.TrainConfig(loss_agg=agg))
        for k in want:
            assert getattr(st, k) == pytest.approx(want[k], rel=1e-15, abs=0), k
    errs = golden("ppo_stats.json")["errors"]
    with pytest.raises(rlo.TrainingError) as e:
        rlo.merge_partials(np.zeros((2, 16)), rlo.TrainConfig())
    assert [3, str(e.value)] == errs["no_tokens"]
    p = np.zeros(16)
    p[6], p[11] = 1, 1
    with pytest.raises(rlo.TrainingError) as e:
        rlo.merge_partials(p, rlo.TrainConfig())
    assert [3, str(e.value)] == errs["nan_adv"]
    p = np.zeros(16)
    p[6], p[0] = 1, np.inf
    with pytest.raises(rlo.TrainingError, match="non-finite loss"):
        rlo.merge_partials(p, rlo.TrainConfig())


def test_merge_partials_token_mean_matches_reference_merge():
    # merge_gradients itself (oracle/_ref) on scalar partials, rank order
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    rng = np.random.default_rng(2)
    for nr in (1, 2, 4):
        parts5 = np.column_stack([rng.standard_normal((nr, 3)), rng.integers(0, 4, nr), rng.integers(4, 9, nr)])
        ref = O.ref_merge_scalars(parts5)
        parts = np.zeros((nr, 16))
        parts[:, [0, 1, 2, 4, 6]] = parts5
        st = rlo.merge_partials(parts, rlo.TrainConfig())
        for k in ("loss", "mean_ratio", "clip_fraction", "mean_kl", "tokens"):
            assert getattr(st, k) == ref[k], k


def test_create_without_gpu_fails_loudly():
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("GPU present")
    with pytest.raises(rlo.CudaError):
        rlo.Objective(0)


def test_policy_worker_rejects_unknown_method():
    from conftest import gpu_available
    if not gpu_available():
        # dispatch validation is host logic; exercise it without a handle
        w = rlo.PolicyWorker.__new__(rlo.PolicyWorker)
        with pytest.raises(rlo.DispatchError, match="unimplemented method 'generate'"):
            rlo.PolicyWorker.call(w, "generate", rlo.Message())


def test_binding_abi_version_matches_header():
    import re
    with open(_abi.HEADER) as f:
        v = int(re.search(r"#define RLO_ABI_VERSION (\d+)", f.read()).group(1))
    assert v == _abi.ABI_VERSION
