"""Small-batch steps: the synchronous path (compute_advantages -> ppo_gradient
-> merge_gradients, host sync each step) vs the same step captured once in a
CUDA graph (merge_gradients_async, result read back with an async copy) and
replayed back to back.  Prints one JSON line per batch shape."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_06122_b200 as rlo  # noqa: E402


def run(B, T, V, iters=200):
    obj = rlo.Objective(0)
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = [torch.empty(B * T, V, device="cuda") for _ in range(3)]
    for m in range(3):
        rlo.synth_logits(x[m], seed=0, model=m)
    K = torch.empty(B, T, dtype=torch.int32, device="cuda")
    rlo.synth_tokens(K, V, seed=0)
    L = torch.full((B,), T, dtype=torch.int32, device="cuda")
    R = torch.rand(B, device="cuda", generator=gen)
    adv = torch.empty(B, T, device="cuda")
    res = torch.zeros(88, dtype=torch.uint8, device="cuda")
    host = torch.zeros(88, dtype=torch.uint8).pin_memory()
    cfg = rlo.TrainConfig(adv_estimator="grpo", group_size=min(B, 8), kl_coef=0.001, kl_estimator="k3")

    def body():
        obj.compute_advantages(cfg, L, T=T, scalar_rewards=R, out=adv)
        obj.ppo_gradient(cfg, K, L, x[0], adv, old_logits=x[1], ref_logits=x[2], outputs=())

    def sync_step():
        body()
        return obj.merge_gradients(cfg)

    for _ in range(5):
        sync_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        sync_step()
    eager_ms = (time.perf_counter() - t0) * 1e3 / iters

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
        obj.merge_gradients_async(cfg, out=res)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        body()
        obj.merge_gradients_async(cfg, out=res)
        host.copy_(res, non_blocking=True)  # the step's result back to the host, inside the graph
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        g.replay()
    torch.cuda.synchronize()
    graph_ms = (time.perf_counter() - t0) * 1e3 / iters
    st = rlo.Objective.step_result(host)
    assert abs(st.loss - sync_step().loss) <= 1e-6 * max(1.0, abs(st.loss))
    tokens = B * T
    print(json.dumps({"B": B, "T": T, "V": V, "P": 3, "eager_ms_per_step": eager_ms, "graph_ms_per_step": graph_ms,
                      "eager_tok_s": tokens / eager_ms * 1e3, "graph_tok_s": tokens / graph_ms * 1e3,
                      "speedup": eager_ms / graph_ms, "launches_per_step": 5}), flush=True)
    obj.close()


if __name__ == "__main__":
    for B, T, V in ((4, 64, 32000), (8, 256, 32000), (64, 512, 32000)):
        run(B, T, V)
