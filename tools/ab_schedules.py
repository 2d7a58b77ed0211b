#!/usr/bin/env python
"""Re-time the best schedules of a bench line with the library's own harness (the bench's
re-timing method: R = 10 windows of >= 200 us of back-to-back launches, verify on), so two
builds of the library can be compared on the same schedules:

    DB200_LIB=/tmp/old/libdroplet_b200.so python tools/ab_schedules.py profiles/bench_r2q_20steps.json
    python tools/ab_schedules.py profiles/bench_r2q_20steps.json

Prints one line per (layer, schedule) and a JSON summary (geomean time per which).
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space, sketches
    from synth import RESNET18, RESNET50, layer_flops, layer_tensors
    from synth.workloads import out_hw

    d = json.load(open(sys.argv[1]))
    which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["dp", "bl"]
    allL = {L["name"]: L for L in RESNET18 + RESNET50}
    dev = torch.device("cuda:0")
    out = []
    for rec in d["per_layer_full"]:
        L = allL[rec["layer"]]
        x, w = layer_tensors(L, 7)
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        P, Q = out_hw(L)
        y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
        shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        pts = []
        for wh in which:
            vals = rec[wh + "_best"]
            for sk in sketches("conv2d", "f32"):
                sp = sketch_space(sk)
                if len(sp) == len(vals) and all(v in sp[i] for i, v in enumerate(vals)):
                    pts.append((wh, (sk, tuple(sp[i].index(v) for i, v in enumerate(vals))), vals))
                    break
        best = min(rec["rt_dp_ns"], rec["rt_bl_ns"])
        num = max(1, int(math.ceil(200000.0 / best)))
        t = Tuner("conv2d", shape, x=xd, w=wd, y=y, seed=1, repeats=10, number=min(num, 4000))
        rs = t.measure([p for _, p, _ in pts])
        for (wh, p, vals), r in zip(pts, rs):
            tf = layer_flops(L) / r.cost_ns / 1e3
            print(f"{rec['layer']:14s} {wh} sk{p[0]} {vals}: {r.cost_ns:8.0f} ns {tf:6.2f} TF/s {r.status} "
                  f"err {r.max_err:.1e}", flush=True)
            out.append({"layer": rec["layer"], "which": wh, "ns": r.cost_ns, "flop": layer_flops(L), "status": r.status})
        t.close()
    summ = {}
    for wh in which:
        xs = [o for o in out if o["which"] == wh and o["status"] == "ok"]
        if xs:
            summ[wh] = {"geomean_ns": math.exp(sum(math.log(o["ns"]) for o in xs) / len(xs)),
                        "agg_tflops": sum(o["flop"] for o in xs) / sum(o["ns"] for o in xs) / 1e3, "n": len(xs)}
    print(json.dumps({"lib": os.environ.get("DB200_LIB", "in-tree"), "summary": summ}))


if __name__ == "__main__":
    main()
