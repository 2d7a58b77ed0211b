#!/usr/bin/env python
"""Where does the ~2 us quantum of event-timed windows come from?  fp32 matmuls (TF32 off) of
growing size; windows (event pairs on the launching stream) around
  A: one graph launch of 1 kernel          B: one graph launch of 8 kernels (/8)
  C: 8 graph launches of 1 kernel (/8)     D: event-record nodes captured inside one graph,
                                              bracketing 1 kernel (events are graph nodes)
The median of 9 windows is printed per mode (us per kernel)."""
import json
import torch


def med(v):
    v = sorted(v)
    return round(v[len(v) // 2], 3)


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for n in range(512, 833, 16):
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        torch.mm(a, b, out=c)
        torch.cuda.synchronize()
        g1, g8 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1, stream=s):
            torch.mm(a, b, out=c)
        with torch.cuda.graph(g8, stream=s):
            for _ in range(8):
                torch.mm(a, b, out=c)
        evd = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(10)]
        gd = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gd, stream=s):
            for i in range(9):
                evd[i].record(s)
                torch.mm(a, b, out=c)
            evd[9].record(s)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(10)]

        def windows(body, per):
            ev[0].record(s)
            for i in range(9):
                body()
                ev[i + 1].record(s)
            torch.cuda.synchronize()
            return [ev[i].elapsed_time(ev[i + 1]) * 1e3 / per for i in range(9)]

        A = windows(lambda: g1.replay(), 1)
        B = windows(lambda: g8.replay(), 8)

        def eight():
            for _ in range(8):
                g1.replay()
        C = windows(eight, 8)
        gd.replay()
        torch.cuda.synchronize()
        D = [evd[i].elapsed_time(evd[i + 1]) * 1e3 for i in range(9)]
        print(json.dumps({"n": n, "A": med(A), "B": med(B), "C": med(C), "D": med(D),
                          "A_all": [round(x, 3) for x in A[:5]], "D_all": [round(x, 3) for x in D[:5]]}), flush=True)


if __name__ == "__main__":
    main()
