"""Top warp-stall sites of an `ncu --page source --csv` export (SASS view): the instructions with
the most stall samples, and the share of samples before the first / after the last instance of
a marker instruction (e.g. FFMA2 for the SIMT kernels, UTCHMMA for tcgen05).

    python tools/ncu_source_summary.py gpurun_out/prof_x.source.csv --marker FFMA2 --top 25
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--marker", default="FFMA2")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    h = rows[1]
    data = rows[2:]
    iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    smp = [int(r[iS]) if r[iS].isdigit() else 0 for r in data]
    tot = sum(smp)
    print(f"kernel: {rows[0][1][:120]}")
    print(f"samples {tot}, SASS instructions {len(data)}")
    idx = [i for i, r in enumerate(data) if a.marker in r[iSrc]]
    if idx:
        pre, mid, post = sum(smp[:idx[0]]), sum(smp[idx[0]:idx[-1] + 1]), sum(smp[idx[-1] + 1:])
        print(f"{a.marker}: {len(idx)} instructions; samples before the first {pre} ({100 * pre / tot:.0f} %), "
              f"between first and last {mid} ({100 * mid / tot:.0f} %), after the last {post} ({100 * post / tot:.0f} %)")
    print("top stall sites (index, samples, SASS):")
    for i in sorted(range(len(data)), key=lambda i: -smp[i])[:a.top]:
        print(f"  {i:5d} {smp[i]:5d}  {data[i][iSrc].strip()[:100]}")


if __name__ == "__main__":
    main()
