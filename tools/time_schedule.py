#!/usr/bin/env python
"""Time one schedule with N back-to-back kernel_run launches between CUDA events.

    python tools/time_schedule.py --layer vgg.512-512@28 --dtype bf16 --values 256,256,128,3,1,32,1 --iters 20
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", required=True)
    ap.add_argument("--values", required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--graph", action="store_true", help="replay a captured CUDA graph of one launch")
    ap.add_argument("--sketch", type=int, default=None)
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
    sk = a.sketch if a.sketch is not None else sketches(L["op"], a.dtype)[0]
    space = sketch_space(sk)
    vals = [int(v) for v in a.values.split(",")]
    p = (sk, tuple(space[d].index(v) for d, v in enumerate(vals)))
    t = Tuner(L["op"], shape, dtype=a.dtype, spaces=[(sk, space)], x=xd, w=wd, y=y, verify=False)
    s = torch.cuda.current_stream()
    for _ in range(3):
        t.run(p, xd, wd, y, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = None
    if a.graph:
        g = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=gs):
            t.run(p, xd, wd, y, stream=gs)
    times = []
    for _ in range(5):
        e0.record(s)
        for _ in range(a.iters):
            if g is not None:
                g.replay()
            else:
                t.run(p, xd, wd, y, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3 / a.iters)
    us = sorted(times)[2]
    print(f"{vals}: {us:.1f} us/launch  {layer_flops(L) / us / 1e6:.1f} TFLOP/s  (all: {[round(v, 1) for v in times]})")


if __name__ == "__main__":
    main()
