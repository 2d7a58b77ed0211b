#!/usr/bin/env python
"""Best schedule per sketch on the same layers: N random valid candidates of each sketch
(same harness, early cut off), printed as one JSON line per (layer, sketch).

    python tools/sketch_compare.py --layers r18 --sketches 1,8 --n 2000
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="r18", help="r18 | r50 | comma list of layer names")
    ap.add_argument("--sketches", default="1,8")
    ap.add_argument("--n", type=int, default=2000)
    ap.add_argument("--top", type=int, default=3)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--early-cut", type=float, default=4.0, help="bench setting; > 0 also enables the precise tier")
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space
    from synth import ALEXNET, BERT, CONFIG1, RESNET18, RESNET50, VGG16, layer_flops, layer_tensors
    from synth.workloads import out_hw

    allL = {L["name"]: L for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT + [CONFIG1]}
    groups = {"r18": RESNET18, "r50": RESNET50, "vgg": VGG16, "alex": ALEXNET, "bert": BERT}
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    if a.layers in groups:
        names = [L["name"] for L in groups[a.layers]]
    else:
        names = a.layers.split(",")
    dev = torch.device("cuda:0")
    for name in names:
        L = allL[name]
        x, w = layer_tensors(L, 1)
        xd, wd = torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt)
        if L["op"] == "conv2d":
            P, Q = out_hw(L)
            y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
            shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        else:
            y = torch.empty((L.get("b", 1), L["m"], L["n"]), device=dev)
            shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
        for sk in [int(s) for s in a.sketches.split(",")]:
            t = Tuner(L["op"], shape, dtype=a.dtype, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y, seed=a.seed,
                      early_cut=a.early_cut)
            smp = t.sample(a.n)
            if not smp:
                print(json.dumps({"layer": name, "sketch": sk, "n": 0}), flush=True)
                t.close()
                continue
            ok = sorted([s for s in smp if s.status == "ok"], key=lambda s: s.cost_ns)
            wrong = sum(s.status == "wrong" for s in smp)
            top = [(t.values(s.point), round(s.cost_ns)) for s in ok[: a.top]]
            best = ok[0].cost_ns if ok else None
            print(json.dumps({"layer": name, "sketch": sk, "n": len(smp), "wrong": wrong, "best_ns": best,
                              "tflops": layer_flops(L) / best / 1e3 if best else None, "top": top}), flush=True)
            t.close()


if __name__ == "__main__":
    main()
