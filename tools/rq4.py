#!/usr/bin/env python
"""RQ4 of the paper: after the same 300 exploration trials, exploit
with Droplet Search vs random sampling, grid search and a genetic algorithm
(AutoTVM's alternatives; the XGBoost tuner needs a learned cost model: out of
scope), 100 trials each, on the same measurement harness; report per layer the
best schedule relative to a 10,000-trial random baseline, trials used and the
exploitation wall time (AlexNet, Droplet ~3x faster).

    python tools/rq4.py --model alexnet --out gpurun_out/rq4.jsonl
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ops", default="conv2d,depthwise_conv2d,dense")
    ap.add_argument("--n-explore", type=int, default=300)
    ap.add_argument("--budget", type=int, default=100)
    ap.add_argument("--baseline", type=int, default=10000)
    ap.add_argument("--early-cut", type=float, default=4.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space
    from synth import layer_tensors, model_layers
    from synth.workloads import out_hw

    dev = torch.device("cuda:0")
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    fout = open(a.out, "a") if a.out else None

    def emit(d):
        s = json.dumps(d)
        print(s, flush=True)
        if fout:
            fout.write(s + "\n")
            fout.flush()

    exploiters = {
        "droplet": lambda t: t.droplet(t.best().point, a.budget)["trials_used"],
        "random": lambda t: len(t.sample(a.budget)),
        "grid": lambda t: len(t.grid(a.budget)),
        "ga": lambda t: len(t.evolve(a.budget)),
    }
    summary = {k: {"wall_s": 0.0, "trials": 0, "ratios": []} for k in exploiters}
    for L in model_layers(a.model, a.batch):
        if L["op"] not in a.ops.split(","):
            continue
        x, w = layer_tensors(L, 0x5EED)
        xd, wd = torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt)
        if L["op"] == "dense":
            yshape, shape = (1, L["m"], L["n"]), {"m": L["m"], "n": L["n"], "k": L["k"]}
        else:
            P, Q = out_hw(L)
            yshape = (L["N"], P, Q, L["K"])
            shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        y = torch.empty(yshape, device=dev)
        spaces = None
        if a.dtype == "bf16" and L["op"] == "conv2d":
            sk = 3 if L["C"] % 8 == 0 else 4
            spaces = [(sk, sketch_space(sk))]
        mk = lambda seed: Tuner(L["op"], shape, dtype=a.dtype, spaces=spaces, x=xd, w=wd, y=y,  # noqa: E731
                                seed=seed, early_cut=a.early_cut)
        t0 = mk(0)
        t0.evolve(a.n_explore)
        explored = [s.point for s in t0.history()]
        t0.close()
        bl = mk(7919)
        bl.sample(a.baseline)
        ref = bl.best().cost_ns
        bl.close()
        rec = {"model": a.model, "layer": L["name"], "op": L["op"], "baseline_best_ns": ref}
        for name, fn in exploiters.items():
            t = mk(1)
            t.measure(explored)  # the same 300 exploration points, re-timed on a fresh history
            before = t.best().cost_ns
            s0 = time.perf_counter()
            used = fn(t)
            el = time.perf_counter() - s0
            best = t.best().cost_ns
            t.close()
            rec[name] = {"best_ns": best, "vs_10k": best / ref, "explore_best_ns": before, "trials": used,
                         "wall_s": el}
            summary[name]["wall_s"] += el
            summary[name]["trials"] += used
            summary[name]["ratios"].append(best / ref)
        emit(rec)
    import math
    out = {"model": a.model, "summary": True}
    for k, v in summary.items():
        r = v["ratios"]
        out[k] = {"geomean_vs_10k": math.exp(sum(math.log(x) for x in r) / len(r)) if r else None,
                  "within_5pct": sum(x <= 1.05 for x in r), "layers": len(r), "trials": v["trials"],
                  "wall_s": v["wall_s"]}
    emit(out)


if __name__ == "__main__":
    main()
