#!/usr/bin/env python
"""Summarise a tools/sweep.py JSONL file as a markdown table (per model + overall)."""
import json
import math
import sys


def main(path):
    rows = [json.loads(l) for l in open(path)]
    S = [r for r in rows if r.get("summary")]
    L = [r for r in rows if not r.get("summary") and "quality" in r]
    print(f"# {path}\n")
    print("| model | tasks | within 5 % of 10k | model time DPAnsor (us) | model time 10k (us) | 10k / DPAnsor time | "
          "tuning wall DPAnsor (s) | tuning wall 10k (s) | wall ratio |")
    print("|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for s in S:
        w = s["tuning_wall_s"]
        print(f"| {s['model']} | {s['tasks']} | {s['within_5pct']} | {s['model_us_dpansor']:.1f} | "
              f"{s['model_us_baseline']:.1f} | {s['speedup_dpansor_vs_baseline']:.3f} | {w['dpansor']:.1f} | "
              f"{w['baseline']:.1f} | {w['ratio']:.1f} |")
    q = [r["quality"] for r in L]
    wd = sum(s["tuning_wall_s"]["dpansor"] for s in S)
    wb = sum(s["tuning_wall_s"]["baseline"] for s in S)
    print(f"\nAll {len(q)} tasks: {sum(x <= 1.05 for x in q)} within 5 % of the 10k baseline; geomean "
          f"DPAnsor/10k cost {math.exp(sum(math.log(x) for x in q) / len(q)):.4f}; worst {max(q):.3f}; "
          f"tuning wall {wd:.0f} s vs {wb:.0f} s ({wb / wd:.1f}x).")
    fr = [r["roofline"]["frac"] for r in L]
    print(f"Roofline fraction of the best schedules: median {sorted(fr)[len(fr) // 2]:.3f}, max {max(fr):.3f}.")


if __name__ == "__main__":
    main(sys.argv[1])
