#!/usr/bin/env python
"""Best fp32 SIMT schedule on large dense GEMMs (no batch-1 latency to speak of): how close the SIMT
families get to the FP32 pipe when parallelism is ample.  300-sample evolution + Droplet per sketch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2406_20037_b200 import Tuner
    dev = torch.device("cuda:0")
    for m, n, k in [(4096, 4096, 4096), (8192, 4096, 1024), (3136 * 8, 64, 576)]:
        x = torch.rand((1, m, k), device=dev) - 0.5
        w = torch.rand((1, n, k), device=dev) - 0.5
        y = torch.empty((1, m, n), device=dev)
        t = Tuner("dense", {"m": m, "n": n, "k": k}, x=x, w=w, y=y, seed=5, early_cut=4.0)
        t.evolve(300)
        best = None
        for sid, _ in t.spaces:
            sb = t.best_of_sketch(sid)
            if sb is not None:
                r = t.droplet(sb.point, 100)
                if best is None or r["best_cost"] < best[0]:
                    best = (r["best_cost"], t.values(r["best"]), r["best"][0])
        tf = 2.0 * m * n * k / best[0] / 1e3
        print(f"dense {m}x{n}x{k}: {best[0] / 1e3:9.1f} us  {tf:6.2f} TFLOP/s ({tf / 73.4:.2f} of FP32 peak)  "
              f"sk{best[2]} {best[1]}", flush=True)
        t.close()


if __name__ == "__main__":
    main()
