#!/usr/bin/env python
"""Key metrics from an `ncu --page raw --csv` export (one profiled launch).

    python tools/ncu_summary.py gpurun_out/prof_tc_vgg512.raw.csv [--flops F] [--bytes B]
"""
import argparse
import csv

KEYS = [
    ("kernel", "Kernel Name"),
    ("duration_us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("smem_dyn_B", "launch__shared_mem_per_block_dynamic"),
    ("dram_read_B", "dram__bytes_read.sum"),
    ("dram_write_B", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fmaheavy_pipe_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"),
    ("inst_fma_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("l2_throughput_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("sm_clock_hz", "smsp__cycles_elapsed.avg.per_second"),
]


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_float(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
             "msecond": 1e3, "nsecond": 1e-3}
    return x * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--flops", type=float, default=None)
    a = ap.parse_args()
    d = load(a.csv)
    out = {}
    for k, m in KEYS:
        if m in d:
            v, u = d[m]
            out[k] = v if k == "kernel" else to_float(v, u)
    for k, v in out.items():
        print(f"{k:24s} {v}")
    if a.flops and out.get("duration_us"):
        print(f"{'TFLOP/s (ncu, cold)':24s} {a.flops / (out['duration_us'] * 1e-6) / 1e12:.1f}")
    if out.get("dram_read_B") is not None and out.get("duration_us"):
        print(f"{'DRAM GB/s':24s} {(out['dram_read_B'] + out['dram_write_B']) / (out['duration_us'] * 1e-6) / 1e9:.0f}")


if __name__ == "__main__":
    main()
