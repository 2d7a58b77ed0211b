#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum launch list by kernel family.

    python tools/summarize_launches.py gpurun_out/launches_r1.csv > profiles/r1_launches.md
"""
import collections
import csv
import io
import sys


def family(name):
    for key in ("simt_gemm_f32_kernel", "simt_pipe_kernel", "direct_conv_kernel", "zero_splitk", "tc_gemm_bf16_kernel", "tc_conv_bf16_kernel", "verify_maxerr", "fp32_peak_kernel",
                "naive_ref_conv", "naive_ref_gemm"):
        if key in name:
            return key
    return name.split("(")[0].replace("void ", "")[:60]


def main(path):
    lines = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        us = v / 1000 if u == "ns" else (v if u in ("us", "usecond") else v * 1000)
        a = agg[family(r["Kernel Name"])]
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list summary: {path}\n")
    print("ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised): compare shares.\n")
    print("| kernel family | launches | total us | share |")
    print("|---|---:|---:|---:|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
