#!/usr/bin/env python
"""Context numbers: cuDNN fp32 (TF32 off) / bf16 time for the bench layers, CUDA events, hot L2.

    python tools/probe_cudnn.py --workload resnet18
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet18")
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    import torch
    import torch.nn.functional as F

    from synth import ALEXNET, BERT, RESNET18, RESNET50, VGG16, layer_flops
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    wl = {"resnet18": RESNET18, "resnet50": RESNET50, "vgg16": VGG16, "alexnet": ALEXNET, "bert": BERT}[a.workload]
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    dev = torch.device("cuda:0")
    for L in wl:
        if L["op"] == "conv2d":
            x = torch.randn(L["N"], L["C"], L["H"], L["W"], device=dev, dtype=dt).to(memory_format=torch.channels_last)
            w = torch.randn(L["K"], L["C"], L["R"], L["S"], device=dev, dtype=dt).to(memory_format=torch.channels_last)
            fn = lambda: F.conv2d(x, w, stride=L["stride"], padding=L["pad"], dilation=L["dil"])  # noqa: E731
        else:
            x = torch.randn(L.get("b", 1), L["m"], L["k"], device=dev, dtype=dt)
            w = torch.randn(L.get("b", 1), L["n"], L["k"], device=dev, dtype=dt)
            fn = lambda: torch.bmm(x, w.transpose(1, 2))  # noqa: E731
        for _ in range(20):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(8):
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6 / 8)
        ts.sort()
        ns = ts[len(ts) // 2]
        print(f"{L['name']:16s} {ns:9.0f} ns  {layer_flops(L) / ns / 1e3:7.2f} TFLOP/s")


if __name__ == "__main__":
    main()
