#!/usr/bin/env python
"""The 20-model layer sweep (BASELINE.json configs[4]): per distinct
tuning task of each model, DPAnsor (300 exploration trials + Droplet <= 100) vs the
10,000-trial random baseline on the same harness, plus the model-level estimate
sum(count x best cost).  One JSON line per task, one summary line per model.

    python tools/sweep.py --models mobilenetv2 --ops depthwise_conv2d
    python tools/sweep.py --models all --dtype f32 --batch 1 --baseline 10000 --out gpurun_out/sweep.jsonl

Roofline per task: conv2d / dense against the FP32 (measured FFMA2 probe) or bf16 (measured)
peak; depthwise conv (no tensor-core shape) against the measured HBM bandwidth,
with algorithmic bytes = |X| + |W| (input dtype) + 4 |Y|.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="all")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ops", default="conv2d,depthwise_conv2d,dense")
    ap.add_argument("--n-sample", type=int, default=300)
    ap.add_argument("--budget", type=int, default=100)
    ap.add_argument("--baseline", type=int, default=10000)
    ap.add_argument("--max-layers", type=int, default=0, help="per model, 0 = all")
    ap.add_argument("--early-cut", type=float, default=2.0, help="R-M3 (as bench.py)")
    ap.add_argument("--repeats", type=int, default=3, help="R-M2: timed windows per candidate (as bench.py)")
    ap.add_argument("--sketch-factor", type=float, default=1.5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    from paper_2406_20037_b200 import Tuner, sketch_space, sketch_valid
    from synth import MODELS, layer_flops, layer_tensors, model_layers
    from synth.workloads import out_hw

    def halo_fits(L):  # sketch 11 has a statically valid point for this layer (as in bench.py)
        import itertools
        if L["C"] % 64 or tuple(L.get("stride", (1, 1))) != (1, 1):
            return False
        shp = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil") if k in L}
        return any(sketch_valid("conv2d", shp, 11, list(v), "bf16") for v in itertools.product(*sketch_space(11)))

    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    from paper_2406_20037_b200 import probe_fp32_peak
    fp32_peak = max(probe_fp32_peak(1)[0] for _ in range(3))  # measured FFMA2 peak (tuner_probe_fp32_peak)
    bf16_peak = float(mp.get("bf16_tflops", 1590.0))
    hbm = float(mp.get("hbm_gbs", 6650.0))
    dev = torch.device("cuda:0")
    tdt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    esz = 4 if a.dtype == "f32" else 2
    ops = set(a.ops.split(","))
    names = list(MODELS) if a.models == "all" else a.models.split(",")
    fout = open(a.out, "a") if a.out else None

    def emit(d):
        s = json.dumps(d)
        print(s, flush=True)
        if fout:
            fout.write(s + "\n")
            fout.flush()

    for mname in names:
        layers = [L for L in model_layers(mname, a.batch) if L["op"] in ops]
        if a.max_layers:
            layers = layers[:a.max_layers]
        tot_dp = tot_bl = wall_dp = wall_bl = 0.0
        within, n_ok = 0, 0
        for L in layers:
            x, w = layer_tensors(L, 0x5EED)
            xd = torch.from_numpy(x).to(dev).to(tdt)
            wd = torch.from_numpy(w).to(dev).to(tdt)
            if L["op"] == "dense":
                yshape = (1, L["m"], L["n"])
                shape = {"m": L["m"], "n": L["n"], "k": L["k"]}
            else:
                P, Q = out_hw(L)
                yshape = (L["N"], P, Q, L["K"])
                shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
            y = torch.empty(yshape, device=dev)
            spaces = None
            if a.dtype == "bf16" and L["op"] == "conv2d":
                sks = ([3 if L["C"] % 8 == 0 else 4] + ([10] if L["C"] <= 16 else [])  # + direct conv (stems)
                       + ([11] if halo_fits(L) else []))  # + halo row tiles where the sketch has valid points
                spaces = [(sk, sketch_space(sk)) for sk in sks]
            fl = layer_flops(L)
            rec = {"model": mname, "layer": L["name"], "op": L["op"], "count": L["count"], "gflop": fl / 1e9,
                   "shape": {k: v for k, v in L.items() if k not in ("name", "count", "op")}}
            t0 = time.perf_counter()
            tu = Tuner(L["op"], shape, dtype=a.dtype, spaces=spaces, x=xd, w=wd, y=y, seed=0,
                       early_cut=a.early_cut, repeats=a.repeats)
            smp = tu.evolve(a.n_sample)
            if not smp:
                rec["skipped"] = "no statically valid schedule"
                emit(rec)
                tu.close()
                continue
            # Droplet from the best point of every sketch within 1.5x of the overall best (R-D17)
            b0 = tu.best()
            starts = [sb for sb in (tu.best_of_sketch(sid) for sid, _ in tu.spaces)
                      if sb is not None and sb.cost_ns <= a.sketch_factor * b0.cost_ns]
            reps = [tu.droplet(sb.point, a.budget) for sb in sorted(starts, key=lambda x: x.cost_ns)]
            rep = min(reps, key=lambda r: r["best_cost"])
            t1 = time.perf_counter()
            bl = Tuner(L["op"], shape, dtype=a.dtype, spaces=spaces, x=xd, w=wd, y=y, seed=7919,
                       early_cut=a.early_cut, repeats=a.repeats)
            bl.sample(a.baseline)
            t2 = time.perf_counter()
            bb = bl.best()
            dp_ns = rep["best_cost"]
            if L["op"] == "depthwise_conv2d":
                byts = esz * (x.size + w.size) + 4 * math.prod(yshape)
                roof = {"bound": "hbm", "achieved": byts / dp_ns, "peak": hbm, "unit": "GB/s"}
            else:
                pk = fp32_peak if a.dtype == "f32" else bf16_peak
                roof = {"bound": "alu" if a.dtype == "f32" else "tensor", "achieved": fl / dp_ns / 1e3, "peak": pk,
                        "unit": "TFLOP/s"}
            roof["frac"] = roof["achieved"] / roof["peak"]
            rec.update(dp_best_ns=dp_ns, dp_best=tu.values(rep["best"]), bl_best_ns=bb.cost_ns,
                       quality=dp_ns / bb.cost_ns, dp_trials=tu.stats()["candidates"],
                       bl_trials=bl.stats()["candidates"], dp_wall_s=t1 - t0, bl_wall_s=t2 - t1, roofline=roof)
            emit(rec)
            tot_dp += L["count"] * dp_ns
            tot_bl += L["count"] * bb.cost_ns
            wall_dp += t1 - t0
            wall_bl += t2 - t1
            within += dp_ns <= 1.05 * bb.cost_ns
            n_ok += 1
            bl.close()
            tu.close()
        emit({"model": mname, "summary": True, "tasks": n_ok, "within_5pct": within,
              "model_us_dpansor": tot_dp / 1e3, "model_us_baseline": tot_bl / 1e3,
              "speedup_dpansor_vs_baseline": tot_bl / max(tot_dp, 1e-9),
              "tuning_wall_s": {"dpansor": wall_dp, "baseline": wall_bl,
                                "ratio": wall_bl / max(wall_dp, 1e-9)}})


if __name__ == "__main__":
    main()
