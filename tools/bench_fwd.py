"""forward_logprobs (policy.cpp:210-233) on one resident micro-batch of
Qwen-vocabulary bf16 rows: kernel time by CUDA events and the HBM rate of its
algorithmic bytes (one read of each row), with and without the entropy.

    python tools/bench_fwd.py [--rows 32768] [--iters 200]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_06122_b200 as rlo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--V", type=int, default=152064)
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    obj = rlo.Objective(0)
    B = args.rows // args.T
    x = torch.empty(args.rows, args.V, dtype=torch.bfloat16, device="cuda")
    rlo.synth_logits(x, seed=0, model=0)
    toks = torch.empty(B, args.T, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(toks, args.V, seed=0)
    L = torch.full((B,), args.T, dtype=torch.int32, device="cuda")
    for ent in (False, True):
        for _ in range(3):
            obj.forward_logprobs(x, toks, L, entropy=ent)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            obj.forward_logprobs(x, toks, L, entropy=ent)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        byts = args.rows * args.V * 2
        print(json.dumps({"row": "forward_logprobs", "entropy": ent, "rows": args.rows, "V": args.V, "ms": ms,
                          "gbs": byts / ms / 1e6, "env": {k: v for k, v in os.environ.items() if k == "RLO_LIB"}}),
              flush=True)


if __name__ == "__main__":
    main()
