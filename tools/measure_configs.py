#!/usr/bin/env python
"""Measure explicit schedules of one layer through the harness and print their costs.

    python tools/measure_configs.py --layer vgg.512-512@28 --dtype bf16 \
        --configs 128,256,64,3,1,32 256,256,64,4,1,32
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--configs", nargs="+", required=True)
    ap.add_argument("--repeats", type=int, default=10)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space, sketches
    from synth import ALEXNET, BERT, CONFIG1, RESNET18, RESNET50, VGG16, layer_flops, layer_tensors
    from synth.workloads import out_hw

    allL = {L["name"]: L for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT + [CONFIG1]}
    L = allL[a.layer]
    dev = torch.device("cuda:0")
    x, w = layer_tensors(L, 1)
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    xd, wd = torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt)
    if L["op"] == "conv2d":
        P, Q = out_hw(L)
        y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
        shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    else:
        y = torch.empty((L.get("b", 1), L["m"], L["n"]), device=dev)
        shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
    sk = sketches(L["op"], a.dtype)[0]
    space = sketch_space(sk)
    t = Tuner(L["op"], shape, dtype=a.dtype, spaces=[(sk, space)], x=xd, w=wd, y=y, repeats=a.repeats)
    pts = []
    for c in a.configs:
        vals = [int(v) for v in c.split(",")]
        vals += [space[d][0] for d in range(len(vals), len(space))]  # omitted trailing knobs: first value
        pts.append((sk, tuple(space[d].index(v) for d, v in enumerate(vals))))
    fl = layer_flops(L)
    for p, r in zip(pts, t.measure(pts)):
        print(f"{t.values(p)} {r.status:6s} {r.cost_ns:10.0f} ns  {fl / max(r.cost_ns, 1e-9) / 1e3:8.1f} TFLOP/s  "
              f"err {r.max_err:.1e}")


if __name__ == "__main__":
    main()
