"""Generator of the explicit-instantiation translation units of the SIMT sketches
(VERDICT r1 housekeeping: the lists were committed without their generator).

    python tools/gen_instantiations.py          # rewrite the files
    python tools/gen_instantiations.py --check  # exit 1 if a committed file differs

kernels/simt_c{0,1}_bm{16,32,64,128}.cu       register-staged SIMT sketch (simt_gemm.cuh): the full
    lattice BN x BK x TT x UNROLL of sketches.cpp's simt_vals for each (CONV, BM); simt_register's
    `if constexpr (simt_static_ok(...))` drops the statically impossible ones at compile time.
kernels/simt_pipe_c{0,1}_bm{16,32,64,128}.cu  cp.async sketch (simt_pipe.cuh): only the lattice
    points that pass pipe_static_ok (threads <= 1024, >= 32 per k group, BK % (4 KW) == 0), so no
    empty registration is emitted.
One TU per (CONV, BM) so nvcc compiles the families in parallel.
"""
import argparse
import os
import sys

KDIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2406_20037_b200", "csrc",
                    "kernels")

BMS = [16, 32, 64, 128]
SIMT = {"BN": [16, 32, 64, 128], "BK": [4, 8, 16, 32], "TT": [2, 4, 8], "UNROLL": [1, 2, 4, 8]}
PIPE = {"BN": [32, 64, 128], "BK": [8, 16, 32], "TT": [2, 4], "KW": [1, 2, 4]}


def pipe_static_ok(bm, bn, bk, tt, kw):  # mirrors simt_pipe.cuh
    return tt <= bm and tt <= bn and (bm // tt) * (bn // tt) >= 32 and (bm // tt) * (bn // tt) * kw <= 1024 \
        and bk % (4 * kw) == 0


def simt_file(conv, bm):
    c = "true" if conv else "false"
    lines = ["// Explicit instantiations of the SIMT fp32 sketch (generated list, one TU per (CONV, BM)",
             "// so nvcc compiles the family in parallel).", '#include "simt_gemm.cuh"', "", "namespace db200 {",
             f"void register_simt_c{int(conv)}_bm{bm}() {{"]
    for bn in SIMT["BN"]:
        for bk in SIMT["BK"]:
            for tt in SIMT["TT"]:
                lines.append("    " + " ".join(f"simt_register<{bm}, {bn}, {bk}, {tt}, {u}, {c}>();"
                                               for u in SIMT["UNROLL"]))
    lines += ["}", "}  // namespace db200", ""]
    return "\n".join(lines)


def pipe_file(conv, bm):
    c = "true" if conv else "false"
    lines = ["// Explicit instantiations of the cp.async multistage SIMT sketch (generated list, one TU",
             "// per (CONV, BM) so nvcc compiles the family in parallel).", '#include "simt_pipe.cuh"', "",
             "namespace db200 {", f"void register_simt_pipe_c{int(conv)}_bm{bm}() {{"]
    for bn in PIPE["BN"]:
        for bk in PIPE["BK"]:
            for tt in PIPE["TT"]:
                for kw in PIPE["KW"]:
                    if pipe_static_ok(bm, bn, bk, tt, kw):
                        lines.append(f"    pipe_register<{bm}, {bn}, {bk}, {tt}, {kw}, {c}>();")
    lines += ["}", "}  // namespace db200", ""]
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    bad = 0
    for conv in (False, True):
        for bm in BMS:
            for name, text in ((f"simt_c{int(conv)}_bm{bm}.cu", simt_file(conv, bm)),
                               (f"simt_pipe_c{int(conv)}_bm{bm}.cu", pipe_file(conv, bm))):
                path = os.path.join(KDIR, name)
                old = open(path).read() if os.path.exists(path) else None
                if a.check:
                    if old != text:
                        print("differs:", name)
                        bad += 1
                elif old != text:
                    with open(path, "w") as f:
                        f.write(text)
                    print("wrote", name)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
