"""Probe: log-softmax error vs a large common logit offset (fp32 rows)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
import paper_2506_06122_b200 as rlo
obj = rlo.Objective(0)
rng = np.random.default_rng(0)
for V in (64, 4096):
    base = (rng.standard_normal(V) * 3).astype(np.float32)
    for off in (0.0, 1e2, 1e3, 1e4, 1e5, -1e2, -1e3, -1e4, -1e5):
        row = (base + np.float32(off)).astype(np.float32)
        tok = int(np.argmax(row))
        x = torch.from_numpy(np.tile(row, (1, 1))).cuda()
        for ent in (False, True):
            out = obj.forward_logprobs(x, torch.tensor([[tok]], dtype=torch.int32, device="cuda"),
                                       torch.tensor([1], dtype=torch.int32, device="cuda"), entropy=ent, token_logit=True)
            lse_gpu = float(out["token_logit"].item()) - float(out["logp"].item())
            lse, _ = O.logsoftmax_row(row.astype(np.float64))
            print(f"V={V} off={off:8.0f} ent={ent}: lp_gpu={out['logp'].item():.7f} lp_ref={float(row[tok])-lse:.7f} "
                  f"err={out['logp'].item() - (float(row[tok])-lse):.3e}")
