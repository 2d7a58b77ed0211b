#!/usr/bin/env python
"""Per-launch floor on this GPU: an empty kernel and a 1-element torch op, 8 back-to-back
launches per CUDA graph, CUDA events (the harness's timing method, DESIGN R-M2)."""
import torch


def time_graph(fn, reps=30):
    for _ in range(5):
        fn()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(8):
                fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 8)
    ts.sort()
    return ts[len(ts) // 2]


x = torch.zeros(1, device="cuda")
y = torch.zeros(1 << 20, device="cuda")
print(f"1-element add_     {time_graph(lambda: x.add_(1)):6.2f} us per launch")
print(f"1M-element add_    {time_graph(lambda: y.add_(1)):6.2f} us per launch")
