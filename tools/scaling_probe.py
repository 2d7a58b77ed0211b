#!/usr/bin/env python
"""How far is a batch-1 fp32 layer from its FMA-bound time?  Tune the same conv at batch
1, 2, 4, 8 (and the dense GEMM of the batch-1 im2col shape) with 300-sample evolution +
Droplet from every sketch's best, and print best time, TFLOP/s and the fixed cost implied by a
linear fit t(b) = t0 + b * t1 (t0 = the per-launch latency floor the batch-1 layer pays).

    python tools/scaling_probe.py --layer r18.l1.3x3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="r18.l1.3x3")
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--n", type=int, default=300)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner
    from synth import RESNET18, RESNET50, layer_flops, layer_tensors
    from synth.workloads import out_hw

    L0 = {L["name"]: L for L in RESNET18 + RESNET50}[a.layer]
    dev = torch.device("cuda:0")

    def tune(op, shape, x, w, y):
        t = Tuner(op, shape, x=x, w=w, y=y, seed=3, early_cut=4.0)
        t.evolve(a.n)
        best = t.best()
        reps = []
        for sid, _ in t.spaces:
            sb = t.best_of_sketch(sid)
            if sb is not None:
                reps.append(t.droplet(sb.point, 100))
        r = min(reps, key=lambda r: r["best_cost"])
        out = (min(best.cost_ns, r["best_cost"]), t.values(r["best"]), r["best"][0])
        t.close()
        return out

    res = []
    for b in [int(v) for v in a.batches.split(",")]:
        L = dict(L0, N=b)
        x, w = layer_tensors(L, 5)
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        P, Q = out_hw(L)
        y = torch.empty((b, P, Q, L["K"]), device=dev)
        shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        ns, vals, sk = tune("conv2d", shape, xd, wd, y)
        f = layer_flops(L)
        res.append((b, ns))
        print(f"conv {a.layer} N={b}: {ns:9.0f} ns {f / ns / 1e3:6.2f} TF/s  sk{sk} {vals}", flush=True)
    # the batch-1 layer as a plain GEMM (im2col shape)
    P, Q = out_hw(L0)
    m, n, k = P * Q, L0["K"], L0["R"] * L0["S"] * L0["C"]
    xd = torch.rand((1, m, k), device=dev) - 0.5
    wd = torch.rand((1, n, k), device=dev) - 0.5
    y = torch.empty((1, m, n), device=dev)
    ns, vals, sk = tune("dense", {"m": m, "n": n, "k": k}, xd, wd, y)
    print(f"dense {m}x{n}x{k}: {ns:9.0f} ns {2 * m * n * k / ns / 1e3:6.2f} TF/s  sk{sk} {vals}", flush=True)
    if len(res) >= 2:
        import numpy as np
        bs = np.array([r[0] for r in res], float)
        ts = np.array([r[1] for r in res], float)
        t1, t0 = np.polyfit(bs, ts, 1)
        print(f"fit t(b) = {t0:.0f} ns + b * {t1:.0f} ns  (FMA-bound per image at the measured peak: "
              f"{layer_flops(L0) / 73.3e3:.0f} ns)")


if __name__ == "__main__":
    main()
