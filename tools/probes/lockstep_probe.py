"""Lockstep streams (RLO_VOCAB_LDG=4) vs sequential: actor log-prob of one bf16 row, P=3, by V."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import oracle as O  # noqa: E402
import paper_2506_06122_b200 as rlo  # noqa: E402

obj = rlo.Objective(0)
for V in (4096, 8192, 16384, 65536, 152064):
    g = torch.Generator().manual_seed(V)
    x = [(torch.randn(4, V, generator=g) * 3).to(torch.bfloat16).cuda() for _ in range(3)]
    toks = torch.zeros(1, 4, dtype=torch.int32, device="cuda")
    L = torch.tensor([4], dtype=torch.int32, device="cuda")
    A = torch.zeros(1, 4, device="cuda")
    res = {}
    for l in ("0", "4"):
        os.environ["RLO_VOCAB_LDG"] = l
        cfg = rlo.TrainConfig()
        o = obj.ppo_gradient(cfg, toks, L, x[0], A, old_logits=x[1], ref_logits=x[2], outputs=("logp", "old_logp", "ref_logp"))
        obj.merge_gradients(cfg)
        res[l] = [o[k].cpu().numpy().ravel() for k in ("logp", "old_logp", "ref_logp")]
    want = [O.logsoftmax_row(x[k][0].float().cpu().numpy().astype(np.float64))[0] for k in range(3)]
    z0 = [float(x[k][0, 0].float()) for k in range(3)]
    print(V, "seq", [round(float(r[0]), 5) for r in res["0"]], "lockstep", [round(float(r[0]), 5) for r in res["4"]],
          "oracle", [round(z0[k] - want[k], 5) for k in range(3)])
