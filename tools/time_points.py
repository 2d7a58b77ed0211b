#!/usr/bin/env python
"""Time chosen schedules of one layer with the library's harness (verify on, R = 10 windows of
>= 200 us of back-to-back launches -- the bench's re-timing method), all in one batch.

    python tools/time_points.py --layer r18.l1.3x3 8:64,64,32,4,1,4,4,6,0,0 8:64,64,32,4,1,4,4,6,0,1
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--window-us", type=float, default=200.0)
    ap.add_argument("--no-verify", action="store_true", help="skip output verification (timing experiments)")
    ap.add_argument("points", nargs="+", help="sketch:v1,v2,...")
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space
    from synth import ALEXNET, BERT, CONFIG1, RESNET18, RESNET50, VGG16, layer_flops, layer_tensors
    from synth.workloads import out_hw

    allL = {L["name"]: L for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT + [CONFIG1]}
    L = dict(allL[a.layer])
    if a.batch:
        L["N" if L["op"] == "conv2d" else "b"] = a.batch
    dev = torch.device("cuda:0")
    x, w = layer_tensors(L, 11)
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    xd, wd = torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt)
    if L["op"] == "conv2d":
        P, Q = out_hw(L)
        y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
        shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    else:
        y = torch.empty((L.get("b", 1), L["m"], L["n"]), device=dev)
        shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
    pts, sks = [], set()
    for s in a.points:
        sk, vals = s.split(":")
        sk = int(sk)
        sp = sketch_space(sk)
        vals = [int(v) for v in vals.split(",")]
        pts.append((sk, tuple(sp[i].index(v) for i, v in enumerate(vals))))
        sks.add(sk)
    spaces = [(sk, sketch_space(sk)) for sk in sorted(sks)]
    # coarse pass to size the windows, then the timed pass
    t0 = Tuner(L["op"], shape, dtype=a.dtype, spaces=spaces, x=xd, w=wd, y=y, seed=1, repeats=3, verify=not a.no_verify)
    coarse = [r.cost_ns for r in t0.measure(pts)]
    t0.close()
    fast = min(c for c in coarse if c > 0 and math.isfinite(c))
    num = max(1, int(math.ceil(a.window_us * 1e3 / fast)))
    t = Tuner(L["op"], shape, dtype=a.dtype, spaces=spaces, x=xd, w=wd, y=y, seed=1, repeats=10,
              number=min(num, 4000), verify=not a.no_verify)
    for s, p, r in zip(a.points, pts, t.measure(pts)):
        tf = layer_flops(L) / r.cost_ns / 1e3 if r.cost_ns > 0 else 0
        print(f"{a.layer} {s:40s} {r.cost_ns:9.0f} ns {tf:7.2f} TF/s {r.status} err {r.max_err:.1e}", flush=True)
    t.close()


if __name__ == "__main__":
    main()
