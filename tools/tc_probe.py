#!/usr/bin/env python
"""Steady-state efficiency of the tcgen05 GEMM sketch on large bf16 GEMMs (no wave
quantisation to speak of): TFLOP/s of chosen schedules, and the best of a short DPAnsor.

    python tools/tc_probe.py --mnk 8192,8192,8192
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mnk", nargs="+", default=["8192,8192,8192", "8192,768,3072", "8192,3072,768"])
    ap.add_argument("--dpansor", type=int, default=120, help="evolve trials before Droplet (0: skip)")
    ap.add_argument("--configs", nargs="*", default=["256,256,64,4,1,0", "256,256,128,3,1,0", "256,128,128,4,1,0",
                                                      "128,256,64,6,1,0", "256,256,64,6,1,1"])
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space
    sp = sketch_space(2)
    for mnk in a.mnk:
        m, n, k = (int(v) for v in mnk.split(","))
        x = torch.randn(1, m, k, device="cuda").to(torch.bfloat16)
        w = torch.randn(1, n, k, device="cuda").to(torch.bfloat16)
        y = torch.empty(1, m, n, device="cuda")
        t = Tuner("dense", {"m": m, "n": n, "k": k}, dtype="bf16", spaces=[(2, sp)], x=x, w=w, y=y, seed=0)
        pts = []
        for c in a.configs:
            vals = [int(v) for v in c.split(",")]
            vals += [sp[d][0] for d in range(len(vals), len(sp))]  # omitted trailing knobs: first value
            p = (2, tuple(sp[d].index(v) for d, v in enumerate(vals)))
            if t.valid(p):
                pts.append(p)
        fl = 2.0 * m * n * k
        for p, r in zip(pts, t.measure(pts)):
            print(f"{mnk:16s} {t.values(p)} {r.status:5s} {r.cost_ns / 1e3:9.1f} us {fl / r.cost_ns / 1e3:7.1f} TFLOP/s")
        if a.dpansor > 0:
            t.evolve(a.dpansor)
            rep = t.droplet(t.best().point, 60)
            print(f"{mnk:16s} DPAnsor best {t.values(rep['best'])} {rep['best_cost'] / 1e3:9.1f} us "
                  f"{fl / rep['best_cost'] / 1e3:7.1f} TFLOP/s")
        t.close()


if __name__ == "__main__":
    main()
