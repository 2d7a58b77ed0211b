#!/usr/bin/env python
"""Best schedule of ONE sketch for a layer (300-sample evolution + Droplet), e.g. to see how far a
sketch that loses the bench's search is from the winner.

    python tools/sketch_best.py --layer r18.conv1 --sketch 9
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", required=True)
    ap.add_argument("--sketch", type=int, required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--n", type=int, default=300)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space
    from synth import ALEXNET, BERT, RESNET18, RESNET50, VGG16, layer_flops, layer_tensors
    from synth.workloads import out_hw
    L = {L["name"]: L for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT}[a.layer]
    dev = torch.device("cuda:0")
    x, w = layer_tensors(L, 3)
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    xd, wd = torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt)
    P, Q = out_hw(L)
    y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
    shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    t = Tuner("conv2d", shape, dtype=a.dtype, spaces=[(a.sketch, sketch_space(a.sketch))], x=xd, w=wd, y=y,
              seed=2, early_cut=4.0)
    t.evolve(a.n)
    r = t.droplet(t.best().point, 100)
    print(f"{a.layer} sketch {a.sketch}: best {r['best_cost']:.0f} ns "
          f"{layer_flops(L) / r['best_cost'] / 1e3:.2f} TFLOP/s {t.values(r['best'])}")
    t.close()


if __name__ == "__main__":
    main()
