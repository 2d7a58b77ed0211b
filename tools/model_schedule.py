"""Model-level DPAnsor in measured mode: Ansor's task scheduler
(tuner_schedule: min(K/L, 64) trials per kernel, then the rest to the kernels with the largest
occurrence x best time, dropping kernels below 1 % of the model, R-F3) spends a budget of K
trials over all distinct kernels of a model; then Droplet Search runs on every kernel from its
best configuration until convergence (<= 100 trials).  The Ansor-10k reference arm spends
10,000 trials with the same scheduler.  Reported per model: the model-level time
sum(count x best cost) after the scheduler, after Droplet, and of the 10k arm; trials and wall
time of both arms; per-task best costs.

    python tools/model_schedule.py --model alexnet --budget 300 --baseline 10000 --out gpurun_out/ms.json
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_tuners(layers, dtype, dev, seed, early_cut):
    import torch
    from paper_2406_20037_b200 import Tuner
    from synth import layer_tensors
    from synth.workloads import out_hw
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    out = []
    for i, L in enumerate(layers):
        x, w = layer_tensors(L, 0x5EED + i)
        xd = torch.from_numpy(x).to(dev).to(tdt)
        wd = torch.from_numpy(w).to(dev).to(tdt)
        if L["op"] == "conv2d":
            P, Q = out_hw(L)
            y = torch.empty((L["N"], P, Q, L["K"]), device=dev)
            shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        else:
            y = torch.empty((L.get("b", 1), L["m"], L["n"]), device=dev)
            shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
        t = Tuner(L["op"], shape, dtype=dtype, x=xd, w=wd, y=y, seed=seed + i, early_cut=early_cut)
        out.append((t, (xd, wd, y)))
    return out


def run(model, batch, dtype, budget, baseline, droplet_budget, early_cut, seed=0):
    import torch
    from paper_2406_20037_b200 import schedule
    from synth import model_layers
    dev = torch.device("cuda:0")
    layers = model_layers(model, batch)
    weights = [float(L.get("count", 1)) for L in layers]
    res = {"model": model, "batch": batch, "dtype": dtype, "tasks": len(layers), "budget": budget,
           "baseline": baseline, "per_task": []}
    # DPAnsor: scheduler with K trials, then Droplet per kernel
    tus = make_tuners(layers, dtype, dev, seed, early_cut)
    t0 = time.perf_counter()
    trials = schedule([t for t, _ in tus], weights, budget)
    t1 = time.perf_counter()
    sched_best = [t.best().cost_ns if t.history() else math.inf for t, _ in tus]
    dp_best, dp_trials = [], []
    for t, _ in tus:
        if not t.history():
            dp_best.append(math.inf)
            dp_trials.append(0)
            continue
        rep = t.droplet(t.best().point, droplet_budget)
        dp_best.append(rep["best_cost"])
        dp_trials.append(rep["trials_used"])
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    # Ansor-10k arm: the same scheduler with the 10,000-trial budget
    bl = make_tuners(layers, dtype, dev, seed + 7919, early_cut)
    t3 = time.perf_counter()
    bl_trials = schedule([t for t, _ in bl], weights, baseline)
    t4 = time.perf_counter()
    bl_best = [t.best().cost_ns if t.history() else math.inf for t, _ in bl]
    model_t = lambda costs: sum(w * c for w, c in zip(weights, costs) if math.isfinite(c))  # noqa: E731
    for i, L in enumerate(layers):
        res["per_task"].append({"task": L["name"], "count": weights[i], "sched_trials": trials[i],
                                "droplet_trials": dp_trials[i], "sched_best_ns": sched_best[i],
                                "dpansor_best_ns": dp_best[i], "bl_trials": bl_trials[i], "bl_best_ns": bl_best[i]})
    res.update({"model_ns_after_scheduler": model_t(sched_best), "model_ns_dpansor": model_t(dp_best),
                "model_ns_ansor10k": model_t(bl_best), "dpansor_over_10k": model_t(dp_best) / model_t(bl_best),
                "wall_s_dpansor": t2 - t0, "wall_s_scheduler": t1 - t0, "wall_s_ansor10k": t4 - t3,
                "trials_dpansor": sum(trials) + sum(dp_trials), "trials_ansor10k": sum(bl_trials)})
    for t, _ in tus + bl:
        t.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--budget", type=int, default=300)
    ap.add_argument("--baseline", type=int, default=10000)
    ap.add_argument("--droplet-budget", type=int, default=100)
    ap.add_argument("--early-cut", type=float, default=4.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    r = run(a.model, a.batch, a.dtype, a.budget, a.baseline, a.droplet_budget, a.early_cut)
    print(json.dumps(r))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
