"""Box probe: device-to-device copy bandwidth (torch), HBM/SM clocks, power."""
import subprocess
import torch
x = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"d2d copy: {2 * x.numel() / ms / 1e6:.0f} GB/s (read+write)")
print(subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm,clocks.max.mem,power.draw,power.limit,temperature.gpu,pci.bus_id",
                      "--format=csv"], capture_output=True, text=True).stdout)

# read-only streaming bandwidth: a reduction over 16 GiB
z = torch.empty(4 << 30, dtype=torch.float32, device="cuda").fill_(1.0)
for _ in range(2):
    z.sum()
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    z.sum()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"read-only (torch sum): {z.numel() * 4 / ms / 1e6:.0f} GB/s")

# our vocab pass (forward_logprobs, P=1) over the same bytes: 131072 rows x V=32000 fp32
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2506_06122_b200 as rlo
obj = rlo.Objective(0)
rows, V = 131072, 32000
lg = z[: rows * V].view(rows, V)
rlo.synth_logits(lg, seed=0, model=0)
toks = torch.zeros(rows // 1024, 1024, dtype=torch.int32, device="cuda")
L = torch.full((rows // 1024,), 1024, dtype=torch.int32, device="cuda")
for ent in (False, True):
    for _ in range(2):
        obj.forward_logprobs(lg, toks, L, entropy=ent)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        obj.forward_logprobs(lg, toks, L, entropy=ent)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"forward_logprobs entropy={ent}: {rows * V * 4 / ms / 1e6:.0f} GB/s")

# bf16 Qwen vocabulary: 32768 rows x 152064
del lg
rows, V = 32768, 152064
lb = z.view(torch.bfloat16)[: rows * V].view(rows, V)
rlo.synth_logits(lb, seed=0, model=0)
toks = torch.zeros(rows // 1024, 1024, dtype=torch.int32, device="cuda")
L = torch.full((rows // 1024,), 1024, dtype=torch.int32, device="cuda")
for ent in (False, True):
    for _ in range(2):
        obj.forward_logprobs(lb, toks, L, entropy=ent)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        obj.forward_logprobs(lb, toks, L, entropy=ent)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"bf16 forward_logprobs entropy={ent}: {rows * V * 2 / ms / 1e6:.0f} GB/s")
