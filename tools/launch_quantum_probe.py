#!/usr/bin/env python
"""Is a back-to-back kernel's duration quantised?  fp32 matmuls (TF32 off) of growing size in a
CUDA graph of 8 launches, timed with events over 20 replays; prints the per-launch time against
the size.  A staircase in ~1 us steps means back-to-back kernels complete on a coarse cadence
(the harness then sees equal costs for kernels whose true durations differ by < 1 us); a smooth
curve means they do not.  Also prints single-launch event windows (event clock resolution)."""
import json
import torch


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    s = torch.cuda.Stream()
    for n in range(256, 1281, 32):
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            torch.mm(a, b, out=c)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(8):
                    torch.mm(a, b, out=c)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        for _ in range(7):
            e0.record(s)
            for _ in range(10):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1) * 1e3 / 80)
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g1, stream=s):
                torch.mm(a, b, out=c)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
        ev[0].record(s)
        for i in range(8):
            g1.replay()
            ev[i + 1].record(s)
        torch.cuda.synchronize()
        singles = [round(ev[i].elapsed_time(ev[i + 1]) * 1e3, 3) for i in range(8)]
        print(json.dumps({"n": n, "us_per_launch": round(sorted(reps)[3], 3), "single_windows_us": singles}),
              flush=True)


if __name__ == "__main__":
    main()
