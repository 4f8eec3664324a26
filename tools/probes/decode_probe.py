"""One decode_sample launch pair (screen + fp64 redo) at the Qwen vocabulary, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2506_06122_b200 as rlo  # noqa: E402

rows, V = int(os.environ.get("ROWS", 32768)), int(os.environ.get("V", 152064))
temp = float(os.environ.get("TEMP", 0.8))
obj = rlo.Objective(0)
x = torch.empty(rows, V, dtype=torch.bfloat16, device="cuda")
rlo.synth_logits(x, seed=1, model=0)
keys = torch.arange(rows, dtype=torch.int64, device="cuda") * 7919
pos = torch.full((rows,), 17, dtype=torch.int64, device="cuda")
for _ in range(3):
    tok, lp = obj.decode_sample(x, temp, 42, 3, keys, pos)
torch.cuda.synchronize()
os.environ["RLO_DECODE_MARGIN"] = "0"
tok64, _ = rlo.Objective(0).decode_sample(x, temp, 42, 3, keys, pos)  # knobs: read at handle creation
print("tokens screened == fp64:", bool((tok == tok64).all().item()), "rows", rows)
# rows the screen leaves to the fp64 kernel
os.environ.pop("RLO_DECODE_MARGIN")
if os.environ.get("MARGIN"):
    os.environ["RLO_DECODE_MARGIN"] = os.environ["MARGIN"]
os.environ["RLO_DECODE_NOREDO"] = "1"
probe = rlo.Objective(0)
for t in (0.6, 0.8, 1.0, 1.3):
    tk, _ = probe.decode_sample(x, t, 42, 3, keys, pos)
    print(f"V={V} T={t} margin={os.environ.get('MARGIN', 'default')}: screen fail rate {(tk < 0).float().mean().item():.3f}")
os.environ.pop("RLO_DECODE_NOREDO")
