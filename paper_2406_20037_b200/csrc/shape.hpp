// shape.hpp — sketch ids and the GEMM view of a problem (kernel-side header).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/tuner.h"

namespace db200 {

enum SketchId : int32_t {
    SK_SIMT_GEMM_F32 = 0,
    SK_SIMT_IGEMM_CONV_F32 = 1,
    SK_TC_GEMM_BF16 = 2,
    SK_TC_IGEMM_CONV_BF16 = 3,
    SK_SIMT_IGEMM_CONV_BF16 = 4,
    SK_SIMT_DWCONV_F32 = 5,
    SK_SIMT_DWCONV_BF16 = 6,
    SK_SIMT_PIPE_GEMM_F32 = 7,
    SK_SIMT_PIPE_CONV_F32 = 8,
    SK_SIMT_DIRECT_CONV_F32 = 9,
    SK_SIMT_DIRECT_CONV_BF16 = 10,
    SK_TC_HALO_CONV_BF16 = 11,
    SK_COUNT = 12
};

// depthwise sketch: shared-memory bytes of a CTA (filters [R*S][ctv] + input window
// [win][ctv], fp32); used by the static validity rule and by the launcher
inline size_t dwconv_smem_bytes(int rs, int ctv, int win) { return (size_t)4 * ((size_t)rs + win) * ctv; }

// tcgen05 sketches: shared memory of the epilogue TMA-store staging (4 warps x 2 boxes x 32 x 32 fp32)
constexpr int kTcEpiBytes = 4 * 2 * 32 * 32 * 4;

// depthwise register-window schedule (ALG 0): taps + two input row segments (one in
// flight) + accumulators must fit the register budget (fp32 values per thread)
constexpr bool dw_win_fits(int vec, int tq, int tp, int ks, int sh) {
    return (ks * ks + 2 * ((tq - 1) * sh + ks) + tp * tq) * vec + ((tq - 1) * sh + ks) <= 90;
}

// cp.async multistage SIMT sketches: shared-memory bytes of a launch (ring of STAGES
// [BM+BN][BK+4] fp32 tiles, or the reduction tile if larger -- KW group partials, or the
// split-K tile staged for 128-bit atomics -- + the conv k table)
// (persistent CTAs: ring + reduction tile side by side, the k table over all of K)
// row stride (floats) of the staged epilogue tile: 8 pad floats put the 4 rows of a warp's
// 8 x 4 thread patch on disjoint banks
constexpr int pipe_red_ld(int bn) { return bn + 8; }
inline size_t pipe_smem_bytes(int bm, int bn, int bk, int kw, int stages, bool conv, int kspan, int vw,
                              int split, int persist = 0) {
    const size_t pipe = (size_t)stages * (bm + bn) * (bk + 4) * 4;
    const size_t red = (kw > 1 || split > 1) ? (size_t)kw * bm * pipe_red_ld(bn) * 4 : 0;
    const size_t ktab = conv ? (size_t)((kspan + vw - 1) / vw) * 8 : 0;
    return (persist ? pipe + red : (pipe > red ? pipe : red)) + ktab;
}
constexpr int kB200Sms = 148;  // static validity rules that depend on the SM count (B200 only)
constexpr int kPipeMaxSlots = 8;  // cp.async slots per thread per operand

// direct conv sketches: the block-size bound of an instantiation (its accumulators need
// registers: KT*TP floats per thread) -- the kernel's __launch_bounds__ and the validity rule
constexpr int direct_max_threads(int kt, int tp) { return kt * tp >= 64 ? 256 : (kt * tp >= 32 ? 512 : 1024); }
// direct conv sketches: filters [R*S*C][BKC] fp32, or (EPI 1) the [PX][BKC + 4] output tile if larger
inline size_t direct_smem_bytes(int rsc, int bkc, int px, int epi) {
    const size_t wb = (size_t)rsc * bkc * 4;
    const size_t yb = epi ? (size_t)px * (bkc + 4) * 4 : 0;
    return wb > yb ? wb : yb;
}

// Stream-K workspace of the tcgen05 sketches (SCHED >= 1): `slots` flags (0 between launches:
// heads re-arm their tails' flags) and one 128 x 256 fp32 partial tile per (group, CTA) slot.
// Owned by a tuner handle and allocated outside graph capture; launches that share one
// workspace must be ordered (one stream), launches of different handles never share one.
struct StreamKScratch {
    unsigned* flags = nullptr;
    float* ws = nullptr;
    int slots = 0;
    int dev = -1;
};

struct ShapeInfo {  // derived GEMM view of the problem (depthwise: M = n*p*q, N = c, K = r*s)
    int32_t op, dtype;
    int64_t batch, M, N, K;     // GEMM: Y[batch][M][N] = A[batch][M][K] * B[batch][N][K]^T
    // conv
    int64_t n, h, w, c, k, r, s, p, q;
    int32_t sh, sw, ph, pw, dh, dw;
    int64_t y_elems, x_elems, w_elems;
};

}  // namespace db200
