"""Out-of-bounds and race checks of our own (compute-sanitizer is closed on the
GPU pool: profiles/r2_sanitizer.txt).

Every input lives between guard regions of NaN (floats / bf16) or sentinel
ids, so a kernel that reads past its rows picks up NaN and fails the oracle
comparison; every output lives between guard regions of a sentinel bit
pattern that must survive the launch (an out-of-bounds write changes it);
row-strided outputs (gradients) also keep their padding columns.  Each launch
runs twice and must give bitwise-identical outputs (a shared-memory or DSMEM
race, or a missing barrier, shows up as run-to-run differences).  Small
shapes, every shipped kernel: the vocab pass (fp32 / bf16, long rows with the
lazy max, lockstep on a deferred offset, unaligned rows), the fused update pass
(cluster + DSMEM), the backward epilogue, the advantage scans, decode."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GUARD = 16384  # elements on each side (64 KB of fp32)
SENT = 0x5A5A5A5A


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2506_06122_b200 as rlo
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch, rlo, rlo.Objective(0)


class Guarded:
    """A device tensor of `shape` in the middle of a buffer whose guard regions
    hold `fill` (inputs: NaN; outputs: the sentinel bit pattern)."""

    def __init__(self, torch, shape, dtype, fill):
        n = int(np.prod(shape))
        self.buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
        if fill == "nan":
            self.buf.fill_(float("nan"))
        else:
            self.buf.view(torch.uint8).fill_(0x5A)
        self.t = self.buf[GUARD:GUARD + n].view(*shape)
        self.torch = torch

    def guards_intact(self):
        g = self.torch.cat([self.buf[:GUARD], self.buf[-GUARD:]]).view(self.torch.uint8)
        return bool((g == 0x5A).all().item())


def guarded_in(torch, a, dtype=None):
    src = torch.from_numpy(np.ascontiguousarray(a))
    g = Guarded(torch, tuple(src.shape), dtype or src.dtype, "nan" if src.dtype.is_floating_point else "sent")
    g.t.copy_(src.to(g.t.dtype).cuda())
    return g.t, g


def guarded_out(torch, shape, dtype):
    return Guarded(torch, shape, dtype, "sent")


def twice(fn):
    """Run fn twice; fn returns a list of output tensors (cloned after each run)."""
    a = [x.clone() for x in fn()]
    b = [x.clone() for x in fn()]
    import torch
    raw = lambda x: x.contiguous().view(-1).view(torch.uint8).cpu().numpy().tobytes()  # noqa: E731
    for x, y in zip(a, b):
        assert raw(x) == raw(y), "outputs differ between two identical launches"
    return a


@pytest.mark.parametrize("dt,V,P", [("f32", 4096, 3), ("f32", 1001, 2), ("bf16", 152064, 3), ("bf16", 4096, 3),
                                    ("bf16", 50257, 1)])
def test_vocab_pass_guards(env, dt, V, P):
    torch, rlo, obj = env
    import ctypes as C

    from paper_2506_06122_b200 import _abi
    from paper_2506_06122_b200.errors import check
    from paper_2506_06122_b200.policy import _batch, _stream
    rng = np.random.default_rng(V + P)
    B, T = 3, 5
    lengths = np.array([5, 2, 4], np.int32)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    rows = [rng.standard_normal((B * T, V)).astype(np.float32) * 3 for _ in range(P)]
    rows[0][4, ::9] = -np.inf
    dev_rows, host_rows = [], []
    for r in rows:
        x, g = guarded_in(torch, r, tdt)
        dev_rows.append(x)
        host_rows.append(x.float().cpu().numpy().astype(np.float32) if dt == "bf16" else r)
    tokens = rng.integers(0, V, (B, T)).astype(np.int32)
    tokens[1, 4] = 10 ** 6  # beyond length 2: never read as a token of a valid row
    K, _ = guarded_in(torch, tokens)
    Lg, _ = guarded_in(torch, lengths)
    adv, _ = guarded_in(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32))
    old = rng.uniform(-9, -1, (B, T)).astype(np.float32)
    OLD, _ = guarded_in(torch, old)
    names = ("logp", "old_logp", "ref_logp", "entropy", "dlogp", "loss", "lse")
    outs = {k: guarded_out(torch, (B, T), torch.float32) for k in names}
    lse64 = guarded_out(torch, (B, T), torch.float64)
    cfg = rlo.TrainConfig(kl_coef=0.01, kl_estimator="k3")

    def run():
        o = _abi.rlo_token_out()
        for k in names:
            setattr(o, k, outs[k].t.data_ptr())
        o.lse64 = lse64.t.data_ptr()
        from paper_2506_06122_b200.policy import _logits
        L = [_logits(x) for x in dev_rows]
        check(_abi.lib().rlo_ppo_gradient(obj._h, C.byref(cfg.to_c()), C.byref(_batch(Lg, K, None, T)),
                                          C.byref(L[0]), C.byref(L[1]) if P > 1 else None,
                                          C.byref(L[2]) if P > 2 else None,
                                          None if P > 1 else C.c_void_p(OLD.data_ptr()),
                                          None if P > 2 else C.c_void_p(OLD.data_ptr()),
                                          C.c_void_p(adv.data_ptr()), C.byref(o), _stream(None, torch.device("cuda"))))
        obj.merge_gradients(cfg)
        return [outs[k].t for k in names] + [lse64.t]

    res = twice(run)
    for k in names:
        assert outs[k].guards_intact(), f"out-of-bounds write next to {k}"
    assert lse64.guards_intact()
    odt = O.F32
    lp, ent, _ = O.forward_logprobs(np.stack(host_rows[0]), odt, V, V, B, T, lengths, tokens)
    m = (np.arange(T)[None, :] < lengths[:, None]).ravel()
    got = res[0].cpu().numpy().ravel()
    assert np.all(np.abs(got[m] - lp[m]) <= 1e-5 * np.maximum(1, np.abs(lp[m]))), "logp (a NaN guard was read?)"
    assert np.all(np.isfinite(res[3].cpu().numpy().ravel()[m])), "entropy"


def test_forward_logprobs_packed_guards(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(3)
    B, T, V = 3, 6, 4096
    lengths = np.array([6, 0, 3], np.int32)
    rows = rng.standard_normal((int(lengths.sum()), V)).astype(np.float32)
    X, _ = guarded_in(torch, rows)
    ss, _ = guarded_in(torch, np.array([0, 6, 6], np.int64))
    toks = rng.integers(0, V, (B, T)).astype(np.int32)
    K, _ = guarded_in(torch, toks)
    Lg, _ = guarded_in(torch, lengths)
    out = twice(lambda: list(obj.forward_logprobs(X, K, Lg, entropy=True, seq_start=ss).values()))
    for b in range(B):
        for t in range(lengths[b]):
            z = rows[[0, 6, 6][b] + t].astype(np.float64)
            lse, _ = O.logsoftmax_row(z)
            want = z[toks[b, t]] - lse
            assert abs(out[0][b, t].item() - want) <= 1e-5 * max(1, abs(want))


@pytest.mark.parametrize("dt,gdt,V", [("f32", "f32", 32000), ("f32", "bf16", 4099), ("bf16", "bf16", 4096)])
def test_backward_and_fused_guards(env, dt, gdt, V):
    """Gradient rows with a padded stride: the padding columns and the guard
    regions keep their sentinel (two-pass backward and the fused cluster pass)."""
    torch, rlo, obj = env
    rng = np.random.default_rng(V)
    B, T = 2, 4
    lengths = np.array([4, 3], np.int32)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    gtdt = torch.float32 if gdt == "f32" else torch.bfloat16
    X, _ = guarded_in(torch, rng.standard_normal((B * T, V)).astype(np.float32) * 2, tdt)
    OLD, _ = guarded_in(torch, rng.standard_normal((B * T, V)).astype(np.float32) * 2, tdt)
    K, _ = guarded_in(torch, rng.integers(0, V, (B, T)).astype(np.int32))
    Lg, _ = guarded_in(torch, lengths)
    A, _ = guarded_in(torch, rng.uniform(-1, 1, (B, T)).astype(np.float32))
    cfg = rlo.TrainConfig(kl_coef=0.0)
    w = obj.loss_weights(cfg, Lg, obj.batch_counts(cfg, Lg, T), T)
    stride = V + 40
    for form in ("two_pass", "fused"):
        G = guarded_out(torch, (B * T, stride), gtdt)

        def run():
            if form == "two_pass":
                o = obj.ppo_gradient(cfg, K, Lg, X, A, old_logits=OLD, outputs=("lse64", "dlogp"))
                obj.merge_gradients(cfg)
                obj.logits_backward(K, Lg, X, o["lse64"], o["dlogp"], w, grad=G.t[:, :V])
            else:
                obj.ppo_gradient_fused(cfg, K, Lg, X, A, w, old_logits=OLD, grad=G.t[:, :V], outputs=())
                obj.merge_gradients(cfg)
            return [G.t[:, :V]]

        twice(run)
        assert G.guards_intact(), form
        pad = G.t[:, V:].contiguous().view(torch.uint8)
        assert bool((pad == 0x5A).all().item()), f"{form}: write into the padding columns of the gradient rows"


def test_advantages_and_decode_guards(env):
    torch, rlo, obj = env
    rng = np.random.default_rng(11)
    B, T = 8, 33
    lengths = rng.integers(0, T + 1, B).astype(np.int32)
    lengths[0] = T
    Lg, _ = guarded_in(torch, lengths)
    M, _ = guarded_in(torch, (rng.random((B, T)) < 0.8).astype(np.uint8))
    R, _ = guarded_in(torch, rng.standard_normal((B, T)).astype(np.float32))
    RS, _ = guarded_in(torch, rng.integers(0, 2, B).astype(np.float32))
    VA, _ = guarded_in(torch, rng.standard_normal((B, T)).astype(np.float32))
    for est in ("reinforce", "gae", "grpo"):
        for wh in (False, True):
            cfg = rlo.TrainConfig(adv_estimator=est, whiten_advantages=wh, group_size=4, gamma=0.97)
            out = guarded_out(torch, (B, T), torch.float32)
            ret = guarded_out(torch, (B, T), torch.float32)

            def run():
                import ctypes as C

                from paper_2506_06122_b200 import _abi
                from paper_2506_06122_b200.errors import check
                from paper_2506_06122_b200.policy import _batch, _stream
                check(_abi.lib().rlo_compute_advantages(
                    obj._h, C.byref(cfg.to_c()), C.byref(_batch(Lg, None, M, T)),
                    None if est == "grpo" else C.c_void_p(R.data_ptr()),
                    C.c_void_p(RS.data_ptr()) if est == "grpo" else None,
                    C.c_void_p(VA.data_ptr()) if est == "gae" else None, C.c_void_p(out.t.data_ptr()),
                    C.c_void_p(ret.t.data_ptr()), _stream(None, torch.device("cuda"))))
                return [out.t, ret.t]

            twice(run)
            assert out.guards_intact() and ret.guards_intact(), (est, wh)
    n, V = 12, 50257
    X, _ = guarded_in(torch, rng.standard_normal((n, V)).astype(np.float32) * 3)
    keys, _ = guarded_in(torch, rng.integers(0, 2**62, n).astype(np.int64))
    pos, _ = guarded_in(torch, np.arange(n, dtype=np.int64))
    for temp in (1.0, 0.8, 1e-7):
        tok = guarded_out(torch, (n,), torch.int32)
        lp = guarded_out(torch, (n,), torch.float32)

        def run():
            import ctypes as C

            from paper_2506_06122_b200 import _abi
            from paper_2506_06122_b200.errors import check
            from paper_2506_06122_b200.policy import _logits, _stream
            check(_abi.lib().rlo_decode_sample(obj._h, C.byref(_logits(X)), n, C.c_double(temp), 3, 1,
                                               C.c_void_p(keys.data_ptr()), C.c_void_p(pos.data_ptr()),
                                               C.c_void_p(tok.t.data_ptr()), C.c_void_p(lp.t.data_ptr()),
                                               _stream(None, torch.device("cuda"))))
            return [tok.t, lp.t]

        got = twice(run)
        assert tok.guards_intact() and lp.guards_intact(), temp
        for i in range(0, n, 3):
            want, _ = O.decode_next(X[i].cpu().numpy().astype(np.float64), temp, 3, 1,
                                    int(keys[i].item()) & (2**64 - 1), i)
            assert got[0][i].item() == want
