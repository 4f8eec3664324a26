"""Actor update step on one GPU: the fused pass (rlo_ppo_gradient_fused: loss +
backward epilogue in one read of the actor logits) against the two-pass form
(rlo_ppo_gradient, then rlo_logits_backward).  Prints one JSON line per
(config, form) with the kernel time and the achieved HBM bandwidth of the
algorithmic bytes (rows*V*(P*s_in + s_grad) fused; rows*V*P*s_in + rows*V*(s_in + s_grad)
two-pass).  Logits are synthetic (include/rlo_synth.h), resident in HBM."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_06122_b200 as rlo  # noqa: E402

CASES = {
    "cfg2": dict(rows=131072, T=1024, V=32000, dt=torch.float32, gdt=torch.float32),
    "cfg3": dict(rows=32768, T=2048, V=152064, dt=torch.bfloat16, gdt=torch.bfloat16),
    "bf16_32k": dict(rows=131072, T=1024, V=32000, dt=torch.bfloat16, gdt=torch.bfloat16),
    "fp32_64k": dict(rows=65536, T=1024, V=65536, dt=torch.float32, gdt=torch.float32),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg2,cfg3")
    ap.add_argument("--P", type=int, default=3)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--forms", default="fused,two_pass")
    args = ap.parse_args()
    obj = rlo.Objective(0)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name in args.cases.split(","):
        c = CASES[name]
        rows, T, V = c["rows"], c["T"], c["V"]
        B = rows // T
        esz, gsz = torch.tensor([], dtype=c["dt"]).element_size(), torch.tensor([], dtype=c["gdt"]).element_size()
        x = [torch.empty(rows, V, dtype=c["dt"], device="cuda") for _ in range(args.P)]
        for m in range(args.P):
            rlo.synth_logits(x[m], seed=0, model=m)
        grad = torch.empty(rows, V, dtype=c["gdt"], device="cuda")
        toks = torch.empty(B, T, dtype=torch.int32, device="cuda")
        rlo.synth_tokens(toks, V, seed=0)
        L = torch.full((B,), T, dtype=torch.int32, device="cuda")
        A = (torch.rand(B, T, device="cuda") * 2 - 1).contiguous()
        OL = torch.full((B, T), -3.0, device="cuda")
        RL = torch.full((B, T), -3.0, device="cuda")
        cfg = rlo.TrainConfig(kl_coef=0.001, kl_estimator="k3")
        kw = {}
        kw.update(old_logits=x[1]) if args.P >= 2 else kw.update(old_logprobs=OL)
        kw.update(ref_logits=x[2]) if args.P >= 3 else kw.update(ref_logprobs=RL)
        cnt = obj.batch_counts(cfg, L, T)
        w = obj.loss_weights(cfg, L, cnt, T)
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

        def fused():
            obj.ppo_gradient_fused(cfg, toks, L, x[0], A, w, grad=grad, outputs=(), **kw)

        def two_pass(t):
            e0, e1, e2 = ev(), ev(), ev()
            e0.record()
            o = obj.ppo_gradient(cfg, toks, L, x[0], A, outputs=("dlogp", "lse"), **kw)
            e1.record()
            obj.logits_backward(toks, L, x[0], o["lse"], o["dlogp"], w, grad=grad)
            e2.record()
            t.append((e0, e1, e2))

        for form in args.forms.split(","):
            for _ in range(2):
                fused() if form == "fused" else two_pass([])
                obj.merge_gradients(cfg)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.iters):
                if form == "fused":
                    e0, e1 = ev(), ev()
                    e0.record()
                    fused()
                    e1.record()
                    ts.append((e0, e1))
                else:
                    two_pass(ts)
                obj.merge_gradients(cfg)
            torch.cuda.synchronize()
            if form == "fused":
                ms = float(np.mean([a.elapsed_time(b) for a, b in ts]))
                byts = rows * V * (args.P * esz + gsz)
                out = {"case": name, "form": form, "P": args.P, "ms": ms, "bytes": byts,
                       "gbs": byts / ms / 1e6, "frac": byts / ms / 1e6 / peak}
            else:
                m1 = float(np.mean([a.elapsed_time(b) for a, b, _ in ts]))
                m2 = float(np.mean([b.elapsed_time(c_) for _, b, c_ in ts]))
                b1, b2 = rows * V * args.P * esz, rows * V * (esz + gsz)
                out = {"case": name, "form": form, "P": args.P, "ms": m1 + m2, "loss_ms": m1, "backward_ms": m2,
                       "bytes": b1 + b2, "gbs": (b1 + b2) / (m1 + m2) / 1e6,
                       "loss_gbs": b1 / m1 / 1e6, "backward_gbs": b2 / m2 / 1e6,
                       "frac": (b1 + b2) / (m1 + m2) / 1e6 / peak}
            out.update(env={k: v for k, v in os.environ.items() if k.startswith("RLO_")})
            print(json.dumps(out), flush=True)
        del x, grad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
