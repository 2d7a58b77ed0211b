#!/usr/bin/env python
"""Harness throughput probe: candidates/s of random sampling on one layer under
different measurement settings, plus the share of candidates cut early.

    python tools/harness_probe.py --layer r18.l2.ds --n 2000
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="r18.l2.ds")
    ap.add_argument("--n", type=int, default=2000)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space, sketches
    from synth import RESNET18, RESNET50, layer_tensors
    from synth.workloads import out_hw

    L = {l["name"]: l for l in RESNET18 + RESNET50}[a.layer]
    dev = torch.device("cuda:0")
    x, w = layer_tensors(L, 1)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    P, Q = out_hw(L)
    y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
    shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
    sk = sketches(L["op"], "f32")[0]
    settings = [
        ("default (W2 R10 cut4)", dict(early_cut=4.0)),
        ("no early cut", dict(early_cut=0.0)),
        ("R5", dict(early_cut=4.0, repeats=5)),
        ("R3 W1", dict(early_cut=4.0, repeats=3, warmup=1)),
        ("cut1.5", dict(early_cut=1.5)),
        ("no verify", dict(early_cut=4.0, verify=False)),
    ]
    for name, kw in settings:
        t = Tuner(L["op"], shape, spaces=[(sk, sketch_space(sk))], x=xd, w=wd, y=y, seed=11, **kw)
        t.sample(64)  # warm: module loads, incumbent
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t.sample(a.n)
        dt = time.perf_counter() - t0
        h = t.history()[64:]
        st = t.stats()
        best = t.best().cost_ns
        cut = sum(1 for s in h if s.status == "ok" and s.cost_ns > kw.get("early_cut", 0) * best) if kw.get("early_cut") else 0
        print(f"{name:24s} {len(h) / dt:8.0f} cand/s  launches/cand {st['kernel_launches'] / max(1, st['candidates']):6.1f}"
              f"  best {best:8.0f} ns  cut~{cut}/{len(h)}")
        t.close()


if __name__ == "__main__":
    main()
