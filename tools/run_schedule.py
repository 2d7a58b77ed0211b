#!/usr/bin/env python
"""Run one schedule of one layer N times through kernel_run (for ncu captures).

    python tools/run_schedule.py --layer r18.l1.3x3 --values 64,64,16,8,1,16 --iters 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="r18.l1.3x3")
    ap.add_argument("--values", required=True, help="comma-separated knob values")
    ap.add_argument("--sketch", type=int, default=None)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--measure", action="store_true")
    ap.add_argument("--model", default=None, help="take --layer from this model's sweep table (synth/models.py)")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space, sketches
    from synth import ALEXNET, BERT, CONFIG1, RESNET18, RESNET50, VGG16, layer_tensors
    from synth.workloads import out_hw

    allL = {L["name"]: L for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT + [CONFIG1]}
    if a.model:
        from synth import model_layers
        allL = {L["name"]: L for L in model_layers(a.model, a.batch)}
    L = allL[a.layer]
    dev = torch.device("cuda:0")
    x, w = layer_tensors(L, 1)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    if a.dtype == "bf16":
        xd, wd = xd.to(torch.bfloat16), wd.to(torch.bfloat16)
    if L["op"] in ("conv2d", "depthwise_conv2d"):
        P, Q = out_hw(L)
        y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
        shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    else:
        y = torch.empty((L.get("b", 1), L["m"], L["n"]), device=dev)
        shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
    sk = a.sketch if a.sketch is not None else sketches(L["op"], a.dtype)[0]
    vals = [int(v) for v in a.values.split(",")]
    space = sketch_space(sk)
    vals += [space[d][0] for d in range(len(vals), len(space))]  # omitted trailing knobs: first value
    idx = tuple(space[d].index(v) for d, v in enumerate(vals))
    t = Tuner(L["op"], shape, dtype=a.dtype, spaces=[(sk, space)], x=xd, w=wd, y=y, verify=a.measure,
              repeats=3, warmup=1)
    if a.measure:  # through the harness: verify run + verify_maxerr + timed graph launches
        r = t.measure([(sk, idx)])[0]
        print("measured", a.layer, vals, r)
        return
    for _ in range(a.iters):
        t.run((sk, idx), xd, wd, y)
    torch.cuda.synchronize()
    print("ran", a.layer, vals, a.iters)


if __name__ == "__main__":
    main()
