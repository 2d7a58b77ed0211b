"""roofline.traffic evidence: DRAM bytes per launch of each timed layer's best schedule.

Step 1 (GPU, under ncu, one process):
    ncu --set full --clock-control none --csv --page raw --log-file gpurun_out/traffic.csv \\
        python tools/capture_traffic.py run --bench profiles/bench_r2.json
  For every layer of the bench run's per_layer_full list, a tuner is created for the layer (its
  naive fp64 reference kernel marks the start of the layer's group in the launch list) and the
  best schedule found by the bench (dp_best) is launched once through kernel_run.
Step 2 (here):
    python tools/capture_traffic.py parse --bench profiles/bench_r2.json --csv gpurun_out/traffic.csv \\
        --out profiles/traffic_r2.json
  sums dram__bytes_read.sum + dram__bytes_write.sum of the schedule's kernels per group (the split-K
  zeroing kernel counts as part of its schedule) and writes {layer: {schedule, dram_bytes, kernels,
  algorithmic_bytes}}; bench.py reads it for roofline.traffic.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def bench_layers(path):
    d = json.load(open(path))
    recs = d.get("per_layer_full") or []
    return [r for r in recs if not r.get("skipped")], d.get("dtype", "f32")


def find_layer(name):
    from synth import ALEXNET, BERT, RESNET18, RESNET50, VGG16
    for L in RESNET18 + RESNET50 + VGG16 + ALEXNET + BERT:
        if L["name"] == name:
            return L
    raise KeyError(name)


def run(args):
    import torch
    import bench
    from paper_2406_20037_b200 import Tuner, sketch_space
    from synth import layer_tensors
    from synth.workloads import out_hw
    recs, dtype = bench_layers(args.bench)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    seen = set()
    for r in recs:
        if r["layer"] in seen:
            continue
        seen.add(r["layer"])
        L = find_layer(r["layer"])
        x, w = layer_tensors(L, 0x5EED)
        xd, wd = torch.from_numpy(x).cuda().to(tdt), torch.from_numpy(w).cuda().to(tdt)
        if L["op"] == "conv2d":
            P, Q = out_hw(L)
            y = torch.empty(L["N"], P, Q, L["K"], device="cuda")
            shape = {k: L[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride", "pad", "dil")}
        else:
            y = torch.empty(L.get("b", 1), L["m"], L["n"], device="cuda")
            shape = {k: L[k] for k in ("b", "m", "n", "k") if k in L}
        sk = r["sketch"]
        vals = r["dp_best"]
        space = sketch_space(sk)
        pt = (sk, tuple(space[d].index(v) for d, v in enumerate(vals)))
        t = Tuner(L["op"], shape, dtype=dtype, spaces=[(sk, space)], x=xd, w=wd, y=y)
        torch.cuda.synchronize()
        t.run(pt, xd, wd, y)
        torch.cuda.synchronize()
        print("captured", r["layer"], sk, vals, flush=True)
        t.close()


def parse(args):
    import bench
    recs, dtype = bench_layers(args.bench)
    lines = open(args.csv).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))  # skip ncu's log lines
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    units = rows[1]
    groups, cur = [], None
    for row in rows[2:]:
        name = row[ix["Kernel Name"]]
        if "naive_ref" in name:
            cur = {"kernels": [], "bytes": 0.0}
            groups.append(cur)
            continue
        if cur is None:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(row[ix[m]].replace(",", "")) * scale.get(units[ix[m]], 1)
        cur["kernels"].append(name.split("(")[0][:80])
        cur["bytes"] += b
    out, layers = {}, []
    for r in recs:
        if r["layer"] not in layers:
            layers.append(r["layer"])
    in_bytes = 4 if dtype == "f32" else 2
    for name, g in zip(layers, groups):
        r = next(x for x in recs if x["layer"] == name)
        out[name] = {"schedule": r["dp_best"], "sketch": r["sketch"], "dram_bytes": g["bytes"],
                     "kernels": g["kernels"], "algorithmic_bytes": bench.layer_min_bytes(find_layer(name), in_bytes)}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    for k, v in out.items():
        print(f"{k:16s} {v['dram_bytes'] / 1e6:8.3f} MB  algorithmic {v['algorithmic_bytes'] / 1e6:8.3f} MB  "
              f"ratio {v['dram_bytes'] / v['algorithmic_bytes']:.2f}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "parse"])
    ap.add_argument("--bench", required=True)
    ap.add_argument("--csv")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "traffic_r2.json"))
    a = ap.parse_args()
    run(a) if a.mode == "run" else parse(a)
