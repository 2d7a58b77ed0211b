#!/usr/bin/env python
"""BASELINE.json configs[0]: dense 512x512x512 fp32 on the 4-knob tile/unroll space (BM, BN, BK,
UNROLL; TT = 4, VEC = 4, STAGES = 2, SPLIT_K = 1 fixed: 256 points, all valid) -- Droplet Search
from the index origin (PLAIN, GROW, RADIUS) against exhaustive brute force on the same harness, on
one GPU.  Each policy runs on a fresh tuner; brute force measures all 256 points on another.  Prints
one JSON line per policy and one for the brute force.

    python tools/config1.py [--early-cut 4]
"""
import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SPACE = [[16, 32, 64, 128], [16, 32, 64, 128], [4, 8, 16, 32], [4], [1, 2, 4, 8], [4], [2], [1]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--early-cut", type=float, default=4.0)
    ap.add_argument("--budget", type=int, default=100)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner
    from synth import layer_tensors
    from synth.workloads import CONFIG1

    m = n = k = 512
    x, w = layer_tensors(CONFIG1, 0)
    dev = torch.device("cuda:0")
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    y = torch.empty(1, m, n, device=dev)
    shape = {"m": m, "n": n, "k": k}
    flops = 2.0 * m * n * k
    pts = [(0, idx) for idx in itertools.product(*[range(len(v)) for v in SPACE])]

    t = Tuner("dense", shape, spaces=[(0, SPACE)], x=xd, w=wd, y=y, early_cut=a.early_cut)
    t0 = time.perf_counter()
    res = t.measure(pts)
    bf_wall = time.perf_counter() - t0
    ok = [r for r in res if r.status == "ok"]
    bf = min(ok, key=lambda r: r.cost_ns)
    print(json.dumps({"config": "dense 512^3 fp32, 4-knob space", "mode": "brute_force", "points": len(pts),
                      "ok": len(ok), "best": t.values(bf.point), "best_ns": bf.cost_ns,
                      "tflops": flops / bf.cost_ns / 1e3, "wall_s": bf_wall}), flush=True)
    t.close()
    for policy in ("plain", "grow", "radius"):
        t = Tuner("dense", shape, spaces=[(0, SPACE)], x=xd, w=wd, y=y, early_cut=a.early_cut, policy=policy)
        t0 = time.perf_counter()
        rep = t.droplet((0, (0,) * 8), a.budget)
        wall = time.perf_counter() - t0
        print(json.dumps({"config": "dense 512^3 fp32, 4-knob space", "mode": f"droplet_{policy}",
                          "start": t.values((0, (0,) * 8)), "best": t.values(rep["best"]),
                          "best_ns": rep["best_cost"], "tflops": flops / rep["best_cost"] / 1e3,
                          "ratio_to_brute_force": rep["best_cost"] / bf.cost_ns,
                          "trials_used": rep["trials_used"], "rounds": rep["rounds"],
                          "converged": rep["converged"], "wall_s": wall}), flush=True)
        t.close()


if __name__ == "__main__":
    main()
