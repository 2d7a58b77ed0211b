"""FP32 pipe peak on this GPU (tuner_probe_fp32_peak): FFMA, FFMA2 and
immediate-form FFMA, each the best of 5 timed launches, repeated `--runs` times.
Writes one JSON object (stdout, and --out)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from paper_2406_20037_b200 import probe_fp32_peak
    torch.cuda.set_device(0)
    res = {"gpu": torch.cuda.get_device_name(0), "sms": torch.cuda.get_device_properties(0).multi_processor_count}
    for mode, name in ((0, "ffma_reg"), (1, "ffma2"), (2, "ffma_imm")):
        v = [probe_fp32_peak(mode)[0] for _ in range(a.runs)]
        res[name] = {"tflops_max": max(v), "tflops_median": statistics.median(v), "runs": v}
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
