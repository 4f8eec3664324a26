"""Vocab pass throughput when rows are not 16-byte aligned (e.g. GPT-2's
V = 50257 in a contiguous bf16 tensor) vs a padded stride."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2506_06122_b200 as rlo  # noqa: E402

obj = rlo.Objective(0)
rows = 32768
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for dt, V, stride in ((torch.bfloat16, 50257, 50257), (torch.bfloat16, 50257, 50264), (torch.float32, 50257, 50257),
                      (torch.float32, 50257, 50260)):
    buf = torch.empty(rows, stride, dtype=dt, device="cuda")
    x = buf[:, :V]
    rlo.synth_logits(x, seed=0, model=0)
    toks = torch.zeros(rows // 1024, 1024, dtype=torch.int32, device="cuda")
    L = torch.full((rows // 1024,), 1024, dtype=torch.int32, device="cuda")
    for ent in (False, True):
        for _ in range(2):
            obj.forward_logprobs(x, toks, L, entropy=ent)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            obj.forward_logprobs(x, toks, L, entropy=ent)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{str(dt).split('.')[-1]} V={V} stride={stride} entropy={ent}: {rows * V * x.element_size() / ms / 1e6:.0f} GB/s")
    del buf
