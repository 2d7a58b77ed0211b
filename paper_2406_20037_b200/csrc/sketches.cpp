// sketches.cpp — the sketch catalogue (Def. 2.1: a sketch is a fixed
// sequence of transformations; its annotations are the knobs) and the static
// validity rules (sketch rules are hardware-dependent; P:596-599:
// schedules that exceed thread limits are invalid).  Host-only.
#include <algorithm>

#include "internal.hpp"

namespace db200 {

static std::vector<SketchDesc> build_catalogue() {
    std::vector<SketchDesc> c;
    // SIMT fp32 GEMM family: block tile BM x BN, K step BK, TT x TT register tile
    // per thread, inner-k UNROLL, split-K (runtime; partial sums reduced with
    // vector atomics into a zeroed Y).
    const std::vector<const char*> simt_names = {"BM", "BN", "BK", "TT", "UNROLL", "VEC", "STAGES", "SPLIT_K"};
    const std::vector<std::vector<int32_t>> simt_vals = {{16, 32, 64, 128}, {16, 32, 64, 128}, {4, 8, 16, 32},
                                                         {2, 4, 8},         {1, 2, 4, 8},       {1, 4},
                                                         {1, 2},            {1, 2, 3, 4, 6, 8, 12, 16}};
    c.push_back({SK_SIMT_GEMM_F32, "simt_gemm_f32", (1 << TUNER_OP_DENSE) | (1 << TUNER_OP_BATCH_MATMUL),
                 TUNER_F32, simt_names, simt_vals});
    c.push_back({SK_SIMT_IGEMM_CONV_F32, "simt_igemm_conv_f32", 1 << TUNER_OP_CONV2D, TUNER_F32, simt_names,
                 simt_vals});
    // cp.async multistage SIMT fp32 family (kernels/simt_pipe.cuh): STAGES-deep cp.async
    // ring with zero-fill gathers, KW warp groups slicing each staged k-tile (summed through
    // shared memory), k-parity FFMA2 accumulators; VEC = cp.async width, SPLIT_K as above.
    // OCC (runtime): 0 = one CTA per work unit (tile x k slice); 2 = two persistent CTAs per SM
    // walking the units, the cp.async ring running on into the next unit's tiles (valid only with
    // more units than CTAs; 1, 3 and 4 per SM were measured and never won, so they are left out
    // of the lattice to keep the 300-trial exploration's space dense).
    // RED (runtime): split-K partial sums by 0 = vector atomics into a zeroed Y, 1 = a cluster of
    // the tile's SPLIT_K CTAs reducing through distributed shared memory (SPLIT_K 2..8, OCC 0).
    const std::vector<const char*> pipe_names = {"BM", "BN", "BK", "TT", "KW", "VEC", "STAGES", "SPLIT_K", "OCC",
                                                 "RED"};
    const std::vector<std::vector<int32_t>> pipe_vals = {{16, 32, 64, 128}, {32, 64, 128}, {8, 16, 32},
                                                         {2, 4},            {1, 2, 4},     {1, 4},
                                                         {2, 3, 4, 6},      {1, 2, 3, 4, 6, 8, 12, 16, 24, 32},
                                                         {0, 2},            {0, 1}};
    c.push_back({SK_SIMT_PIPE_GEMM_F32, "simt_pipe_gemm_f32", (1 << TUNER_OP_DENSE) | (1 << TUNER_OP_BATCH_MATMUL),
                 TUNER_F32, pipe_names, pipe_vals});
    c.push_back({SK_SIMT_PIPE_CONV_F32, "simt_pipe_conv_f32", 1 << TUNER_OP_CONV2D, TUNER_F32, pipe_names,
                 pipe_vals});
    // tcgen05 bf16 GEMM family: UMMA tile BM x BN (accumulator in TMEM), K step
    // BK staged by TMA with 128-byte swizzle, STAGES-deep mbarrier pipeline,
    // split-K (runtime).
    // BM = 256 is the CTA-pair schedule (cta_group::2, UMMA M = 256 over two SMs);
    // SCHED 0 = persistent tile loop (+ split-K), 1 = stream-K (equal share of all k-blocks),
    // 2 = whole waves tile by tile + the remainder tiles cut into k-chunks, one per group.
    // RASTER (runtime): the order tiles are handed to the persistent CTAs, 0 = M fastest
    // (concurrent CTAs share the B panel), 1 = N fastest (they share the A panel).
    // EPI (runtime): how the epilogue writes the fp32 tile, both staged through 128B-swizzled shared
    // memory: 1 = TMA stores (cp.async.bulk.tensor), 2 = coalesced 128-byte st.global segments.
    // (Unstaged 128-bit stores straight from the TMEM registers were measured 7-50 % slower on
    // every layer tried, the smem-bound N = 64 halo tiles included, and are not in the lattice.)
    // EW (compiled): epilogue warps, 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each
    // draining every other 32-column chunk).
    const std::vector<const char*> tc_names = {"BM", "BN", "BK", "STAGES", "SPLIT_K", "SCHED", "RASTER", "EPI", "EW"};
    // STAGES and SPLIT_K are runtime knobs (the ring depth sizes dynamic shared memory).  RASTER:
    // 0 = M fastest, 1 = N fastest, 2 / 3 = bands of 8 M / N tiles (L2 reuse of both panels).
    const std::vector<std::vector<int32_t>> tc_vals = {{128, 256}, {64, 128, 192, 256}, {64, 128},
                                                       {2, 3, 4, 5, 6, 7, 8}, {1, 2, 3, 4, 6, 8}, {0, 1, 2},
                                                       {0, 1, 2, 3},          {1, 2},       {4, 8}};
    c.push_back({SK_TC_GEMM_BF16, "tc_gemm_bf16", (1 << TUNER_OP_DENSE) | (1 << TUNER_OP_BATCH_MATMUL), TUNER_BF16,
                 tc_names, tc_vals});
    // implicit-GEMM conv: the 128-row M tile is a (128/TILE_Q) x TILE_Q rectangle of output pixels
    const std::vector<const char*> tcc_names = {"BM",     "BN",    "BK",     "STAGES", "SPLIT_K",
                                                "TILE_Q", "SCHED", "RASTER", "EPI",    "EW"};
    std::vector<std::vector<int32_t>> tcc_vals(tc_vals.begin(), tc_vals.end() - 4);
    tcc_vals.push_back({8, 16, 32});
    tcc_vals.push_back({0, 1, 2});
    tcc_vals.push_back({0, 1, 2, 3});
    tcc_vals.push_back({1, 2});
    tcc_vals.push_back({4, 8});
    c.push_back({SK_TC_IGEMM_CONV_BF16, "tc_igemm_conv_bf16", 1 << TUNER_OP_CONV2D, TUNER_BF16, tcc_names,
                 tcc_vals});
    // halo row tiles (a sketch of its own: a different loop structure, not a TILE_Q value -- its
    // points would be a sliver of sketch 3's space, rarely drawn and unreachable by coordinate
    // descent from it): stride-1 convs, a tile is 128 output pixels of one row; the R input-row
    // windows of 128 + S - 1 pixels it needs sit in a ring of STAGES row slots and filter tap
    // (r, s) is the row-shifted UMMA view of window r.  A CTA runs down the output rows, so each
    // tile loads ONE new input row (not R*S shifted copies) and the weights stay resident.
    const std::vector<const char*> tch_names = {"BM", "BN", "STAGES", "EPI", "EW"};
    const std::vector<std::vector<int32_t>> tch_vals = {{128, 256}, {64, 128, 192, 256}, {2, 3, 4, 5, 6, 7, 8},
                                                        {1, 2},     {4, 8}};
    c.push_back({SK_TC_HALO_CONV_BF16, "tc_halo_conv_bf16", 1 << TUNER_OP_CONV2D, TUNER_BF16, tch_names, tch_vals});
    // the SIMT implicit-GEMM sketch on bf16 inputs (widened to fp32 at staging, fp32
    // accumulate): a second bf16 conv sketch, and the only one for C % 8 != 0 (TMA needs
    // 16-byte strides); a restricted compile-time lattice
    const std::vector<std::vector<int32_t>> simt16_vals = {{16, 32, 64, 128}, {16, 32, 64, 128}, {8, 16, 32},
                                                           {4, 8},            {1, 4},             {1, 4},
                                                           {1, 2},            {1, 2, 3, 4, 6, 8, 12, 16}};
    c.push_back({SK_SIMT_IGEMM_CONV_BF16, "simt_igemm_conv_bf16", 1 << TUNER_OP_CONV2D, TUNER_BF16, simt_names,
                 simt16_vals});
    // direct conv (SURVEY §8(d).1 `simt_direct_conv`) for few-input-channel layers: KT output
    // channels per thread (compile-time), PX pixels x BKC channels per CTA, EPI 0 per-thread
    // stores / 1 tile staged through shared memory (runtime)
    const std::vector<const char*> dc_names = {"KT", "TP", "PX", "BKC", "EPI"};
    const std::vector<std::vector<int32_t>> dc_vals = {{4, 8, 16, 32, 64}, {1, 2, 4}, {32, 64, 128, 256},
                                                       {16, 32, 64, 128}, {0, 1}};
    c.push_back({SK_SIMT_DIRECT_CONV_F32, "simt_direct_conv_f32", 1 << TUNER_OP_CONV2D, TUNER_F32, dc_names, dc_vals});
    c.push_back({SK_SIMT_DIRECT_CONV_BF16, "simt_direct_conv_bf16", 1 << TUNER_OP_CONV2D, TUNER_BF16, dc_names,
                 dc_vals});
    // depthwise conv: VEC channels per thread (vector loads along C), CT
    // threads across channels, TQ output columns per thread, QT x PT threads across
    // output columns / rows, TP output rows per thread, ALG = 0 register window,
    // 1 shared-memory window, 2 L1 taps (ALG 1 / 2: TP = 1)
    const std::vector<const char*> dw_names = {"VEC", "CT", "TQ", "QT", "PT", "TP", "ALG"};
    const std::vector<std::vector<int32_t>> dw_vals = {{1, 2, 4}, {8, 16, 32, 64}, {1, 2, 4}, {1, 2, 4, 8},
                                                       {1, 2, 4, 8}, {1, 2, 4}, {0, 1, 2}};
    c.push_back({SK_SIMT_DWCONV_F32, "simt_dwconv_f32", 1 << TUNER_OP_DEPTHWISE_CONV2D, TUNER_F32, dw_names,
                 dw_vals});
    c.push_back({SK_SIMT_DWCONV_BF16, "simt_dwconv_bf16", 1 << TUNER_OP_DEPTHWISE_CONV2D, TUNER_BF16, dw_names,
                 dw_vals});
    return c;
}

static const std::vector<SketchDesc>& catalogue() {
    static const std::vector<SketchDesc> c = build_catalogue();
    return c;
}

const SketchDesc* sketch_desc(int32_t id) {
    for (const auto& d : catalogue())
        if (d.id == id) return &d;
    return nullptr;
}

bool make_shape_info(int32_t op, const tuner_shape& s, ShapeInfo& o, std::string& why) {
    o = ShapeInfo{};
    o.op = op;
    o.dtype = s.dtype;
    if (s.dtype != TUNER_F32 && s.dtype != TUNER_BF16) { why = "unknown dtype"; return false; }
    if (op == TUNER_OP_DENSE || op == TUNER_OP_BATCH_MATMUL) {
        o.batch = op == TUNER_OP_DENSE ? 1 : s.b;
        o.M = s.m; o.N = s.n; o.K = s.k;
        if (o.batch < 1 || o.M < 1 || o.N < 1 || o.K < 1) { why = "b, m, n, k must be >= 1"; return false; }
        o.x_elems = o.batch * o.M * o.K;
        o.w_elems = o.batch * o.N * o.K;
        o.y_elems = o.batch * o.M * o.N;
        return true;
    }
    if (op != TUNER_OP_CONV2D && op != TUNER_OP_DEPTHWISE_CONV2D) { why = "unknown op"; return false; }
    if (s.N < 1 || s.C < 1 || s.H < 1 || s.W < 1 || s.K < 1 || s.R < 1 || s.S < 1) {
        why = "conv N, C, H, W, K, R, S must be >= 1"; return false;
    }
    if (s.stride_h < 1 || s.stride_w < 1 || s.dil_h < 1 || s.dil_w < 1 || s.pad_h < 0 || s.pad_w < 0) {
        why = "stride/dilation must be >= 1 and padding >= 0"; return false;
    }
    o.n = s.N; o.h = s.H; o.w = s.W; o.c = s.C; o.k = s.K; o.r = s.R; o.s = s.S;
    o.sh = s.stride_h; o.sw = s.stride_w; o.ph = s.pad_h; o.pw = s.pad_w; o.dh = s.dil_h; o.dw = s.dil_w;
    o.p = (s.H + 2 * s.pad_h - s.dil_h * (s.R - 1) - 1) / s.stride_h + 1;
    o.q = (s.W + 2 * s.pad_w - s.dil_w * (s.S - 1) - 1) / s.stride_w + 1;
    if (o.p < 1 || o.q < 1) { why = "empty conv output"; return false; }
    o.batch = 1;
    o.M = o.n * o.p * o.q;
    o.N = o.k;
    o.x_elems = o.n * o.h * o.w * o.c;
    if (op == TUNER_OP_DEPTHWISE_CONV2D) {  // groups = C = K (R-C5): W is [C][R][S]
        if (s.K != s.C) { why = "depthwise_conv2d needs K == C"; return false; }
        o.K = o.r * o.s;
        o.w_elems = o.c * o.r * o.s;
    } else {
        o.K = o.r * o.s * o.c;
        o.w_elems = o.k * o.r * o.s * o.c;
    }
    o.y_elems = o.M * o.N;
    if (o.M >= (1ll << 31) || o.K >= (1ll << 31) || o.N >= (1ll << 31)) { why = "problem too large"; return false; }
    return true;
}

static bool simt_valid(const ShapeInfo& sh, const int32_t* v) {
    const int bm = v[0], bn = v[1], bk = v[2], tt = v[3], vec = v[5], split = v[7];
    if (tt > bm || tt > bn) return false;
    const int threads = (bm / tt) * (bn / tt);
    if (threads > 1024 || threads < 1) return false;
    const int la = (bm * (bk / 4) + threads - 1) / threads;  // float4 staging slots per thread
    const int lb = (bn * (bk / 4) + threads - 1) / threads;
    if (4 * (la + lb) > 64) return false;  // register budget for the staging buffers
    // 128-bit loads need 4 consecutive k inside one row / one (r,s) tap
    if (vec == 4 && (sh.op == TUNER_OP_CONV2D ? (sh.c % 4) : (sh.K % 4)) != 0) return false;
    const int64_t ktiles = (sh.K + bk - 1) / bk;
    if (split > ktiles) return false;  // empty K slices
    if ((split - 1) * ((ktiles + split - 1) / split) >= ktiles) return false;  // a CTA slice would be empty
    const int64_t ntiles = (sh.N + bn - 1) / bn;
    if (ntiles > 65535 || (int64_t)split * sh.batch > 65535) return false;
    // the conv gather keeps the image base offset n*H*W*C in 32-bit int
    if (sh.op == TUNER_OP_CONV2D && sh.x_elems >= (1ll << 31)) return false;
    return true;
}

static bool pipe_valid(const ShapeInfo& sh, const int32_t* v) {
    const int bm = v[0], bn = v[1], bk = v[2], tt = v[3], kw = v[4], vec = v[5], stages = v[6], split = v[7],
              occ = v[8], red = v[9];
    if (red == 1 && (split < 2 || split > 8 || occ != 0)) return false;  // a portable cluster of the k slices
    const bool conv = sh.op == TUNER_OP_CONV2D;
    if (tt > bm || tt > bn) return false;
    const int gt = (bm / tt) * (bn / tt), threads = gt * kw;
    if (gt < 32 || threads > 1024 || bk % (4 * kw)) return false;
    if (vec == 4 && (conv ? (sh.c % 4) : (sh.K % 4)) != 0) return false;  // 16-byte cp.async inside one tap / row
    const int chunks = (bm > bn ? bm : bn) * (bk / vec);
    if ((chunks + threads - 1) / threads > kPipeMaxSlots) return false;  // cp.async slots per thread
    const int64_t ktiles = (sh.K + bk - 1) / bk;
    if (split > ktiles) return false;
    if ((split - 1) * ((ktiles + split - 1) / split) >= ktiles) return false;  // a CTA slice would be empty
    const int64_t kspan = ((ktiles + split - 1) / split) * bk;
    if (pipe_smem_bytes(bm, bn, bk, kw, stages, conv, (int)kspan, vec, split) > 227 * 1024) return false;
    if (occ > 0) {  // persistent: only when there are more units than CTAs (else = OCC 0)
        const int64_t units = ((sh.M + bm - 1) / bm) * ((sh.N + bn - 1) / bn) * sh.batch * split;
        if (units <= (int64_t)occ * kB200Sms) return false;
        if (pipe_smem_bytes(bm, bn, bk, kw, stages, conv, (int)(ktiles * bk), vec, split, 1) > 227 * 1024)
            return false;
    }
    const int64_t ntiles = (sh.N + bn - 1) / bn;
    if (ntiles > 65535 || (int64_t)split * sh.batch > 65535) return false;
    if (conv && (sh.r - 1) * sh.dh >= 32767) return false;  // tap offsets packed in 16 bits
    // the kernel forms element offsets (m * K, row * K, the conv image base) in 32-bit int
    if (sh.x_elems >= (1ll << 31) || sh.w_elems >= (1ll << 31)) return false;
    return true;
}

static bool direct_valid(const ShapeInfo& sh, const int32_t* v) {
    const int kt = v[0], tp = v[1], px = v[2], bkc = v[3], epi = v[4];
    if (sh.c > 16) return false;  // sketch rule: the direct loop nest is for few-channel stems
    if (kt > bkc || bkc % kt || kt * tp > 64) return false;
    const int threads = px * (bkc / kt);
    if (threads < 32 || threads > direct_max_threads(kt, tp)) return false;
    if (direct_smem_bytes((int)(sh.r * sh.s * sh.c), bkc, px * tp, epi) > 227 * 1024) return false;
    if ((sh.k + bkc - 1) / bkc > 65535) return false;
    return true;
}

static bool tc_valid(const ShapeInfo& sh, const int32_t* v) {
    const int bm = v[0], bn = v[1], bk = v[2], stages = v[3], split = v[4];
    const int sched = sh.op == TUNER_OP_CONV2D ? v[6] : v[5];
    if (sh.dtype != TUNER_BF16) return false;
    if (sched >= 1 && split != 1) return false;  // stream-K already splits the reduction
    // TMA needs 16-byte aligned global strides: K (bf16) multiple of 8.
    int64_t ktiles;
    if (sh.op == TUNER_OP_CONV2D) {
        const int tq = v[5], tp = 128 / tq;
        if (sh.c % 8) return false;
        if (sh.sh > 8 || sh.sw > 8) return false;                  // TMA traversal stride <= 8
        if (tq * sh.sw > 256 || tp * sh.sh > 256) return false;    // TMA box extent <= 256
        if (bk > 64 && sh.c < bk) return false;                    // a fully zero channel block
        ktiles = sh.r * sh.s * ((sh.c + bk - 1) / bk);
    } else {
        if (sh.K % 8) return false;
        ktiles = (sh.K + bk - 1) / bk;
    }
    if (bn > 256 || (bm != 128 && bm != 256)) return false;
    const int cg = bm / 128;  // CTAs per tile: each stages 128 rows of A and bn/cg rows of B
    const int64_t smem = (int64_t)stages * (128 + bn / cg) * bk * 2 + 1024 /*align*/ + 256 /*barriers*/ +
                         kTcEpiBytes /*epilogue staging*/;
    if (smem > 227 * 1024) return false;
    if (split > ktiles) return false;
    if ((int64_t)split * sh.batch > 65535) return false;
    return true;
}

static bool halo_valid(const ShapeInfo& sh, const int32_t* v) {
    const int bm = v[0], bn = v[1], stages = v[2];
    if (sh.dtype != TUNER_BF16 || sh.op != TUNER_OP_CONV2D) return false;
    // stride 1, no dilation, whole 64-channel blocks (TMA boxes of 128 B rows)
    if (sh.sh != 1 || sh.sw != 1 || sh.dh != 1 || sh.dw != 1 || sh.c % 64 || sh.k % 4) return false;
    if (128 + sh.s - 1 > 256) return false;  // a window is one TMA box (extent <= 256)
    if (stages < sh.r + 1) return false;     // STAGES = window slots: R rows + >= 1 prefetched
    if (bn > 256 || (bm != 128 && bm != 256)) return false;
    const int cg = bm / 128;
    const int64_t cb = sh.c / 64;
    const int64_t win = ((128 + sh.s - 1) * 128 + 1023) / 1024 * 1024;
    const int64_t bres = cb * sh.r * sh.s * (bn / cg) * 64 * 2;  // every tap's B slice, resident
    const int64_t smem = 1024 + (int64_t)stages * cb * win + bres + kTcEpiBytes + 256;
    return smem <= 227 * 1024 && (sh.k + bn - 1) / bn <= 65535;
}

static bool dw_valid(const ShapeInfo& sh, const int32_t* v) {
    const int vec = v[0], ct = v[1], tq = v[2], qt = v[3], pt = v[4], tp = v[5], alg = v[6];
    const int threads = ct * qt * pt;
    if (threads < 32 || threads > 512) return false;  // __launch_bounds__(512): no spills
    if (sh.c % vec) return false;                     // aligned vector loads along C
    if (alg == 0) {  // register window: compiled for 3x3 / 5x5, stride 1 / 2, no dilation
        if (sh.r != sh.s || (sh.r != 3 && sh.r != 5) || sh.sh != sh.sw || sh.sh > 2 || sh.dh != 1 || sh.dw != 1)
            return false;
        if (!dw_win_fits(vec, tq, tp, (int)sh.r, sh.sh)) return false;  // taps + row segment + accumulators
    } else {
        if (tp != 1) return false;
        const int64_t ih = (int64_t)(pt - 1) * sh.sh + (sh.r - 1) * sh.dh + 1;
        const int64_t iw = (int64_t)(qt * tq - 1) * sh.sw + (sh.s - 1) * sh.dw + 1;
        const size_t bytes = dwconv_smem_bytes((int)(sh.r * sh.s), ct * vec, alg == 1 ? (int)(ih * iw) : 0);
        if (bytes > 227 * 1024) return false;
    }
    const int64_t tiles_p = (sh.p + pt * tp - 1) / (pt * tp);
    if (sh.n * tiles_p > 65535 || (sh.q + qt * tq - 1) / (qt * tq) > 65535) return false;
    return true;
}

bool sketch_valid(int32_t id, const ShapeInfo& sh, const int32_t* v) {
    const SketchDesc* d = sketch_desc(id);
    if (!d || !(d->op_mask & (1 << sh.op)) || d->dtype != sh.dtype) return false;
    switch (id) {
        case SK_SIMT_GEMM_F32:
        case SK_SIMT_IGEMM_CONV_F32:
        case SK_SIMT_IGEMM_CONV_BF16: return simt_valid(sh, v);
        case SK_SIMT_PIPE_GEMM_F32:
        case SK_SIMT_PIPE_CONV_F32: return pipe_valid(sh, v);
        case SK_SIMT_DIRECT_CONV_F32:
        case SK_SIMT_DIRECT_CONV_BF16: return direct_valid(sh, v);
        case SK_TC_GEMM_BF16:
        case SK_TC_IGEMM_CONV_BF16: return tc_valid(sh, v);
        case SK_SIMT_DWCONV_F32:
        case SK_SIMT_DWCONV_BF16: return dw_valid(sh, v);
        case SK_TC_HALO_CONV_BF16: return halo_valid(sh, v);
        default: return false;
    }
}

}  // namespace db200

// ---------------------------------------------------------------- C ABI (catalogue)
using namespace db200;

extern "C" tuner_status tuner_sketches(int32_t op, int32_t dtype, int32_t* ids, int32_t cap, int32_t* n_out) {
    if (!n_out) return fail(TUNER_EINVAL, "n_out is NULL");
    int32_t n = 0;
    for (const auto& d : catalogue()) {
        if ((d.op_mask & (1 << op)) && d.dtype == dtype) {
            if (ids && n < cap) ids[n] = d.id;
            ++n;
        }
    }
    *n_out = n;
    return TUNER_OK;
}

extern "C" tuner_status tuner_sketch_space(int32_t sketch, int32_t* nknobs, int32_t* card, int32_t* values) {
    const SketchDesc* d = sketch_desc(sketch);
    if (!d) return fail(TUNER_ERANGE, "unknown sketch id");
    if (!nknobs || !card || !values) return fail(TUNER_EINVAL, "NULL output");
    *nknobs = (int32_t)d->values.size();
    int32_t off = 0;
    for (size_t i = 0; i < d->values.size(); ++i) {
        card[i] = (int32_t)d->values[i].size();
        for (int32_t v : d->values[i]) values[off++] = v;
    }
    return TUNER_OK;
}

extern "C" const char* tuner_sketch_name(int32_t sketch) {
    const SketchDesc* d = sketch_desc(sketch);
    return d ? d->name : nullptr;
}

extern "C" const char* tuner_knob_name(int32_t sketch, int32_t knob) {
    const SketchDesc* d = sketch_desc(sketch);
    if (!d || knob < 0 || knob >= (int32_t)d->knob_names.size()) return nullptr;
    return d->knob_names[knob];
}

extern "C" tuner_status tuner_sketch_valid(int32_t op, const tuner_shape* shape, int32_t sketch, const int32_t* values,
                                           int32_t nvalues, int32_t* valid) {
    if (!shape || !values || !valid) return fail(TUNER_EINVAL, "NULL argument");
    const SketchDesc* d = sketch_desc(sketch);
    if (!d) return fail(TUNER_ERANGE, "unknown sketch id");
    if (nvalues != (int32_t)d->values.size()) return fail(TUNER_EDIM, "one value per knob of the sketch");
    ShapeInfo sh;
    std::string why;
    if (!make_shape_info(op, *shape, sh, why)) return fail(TUNER_EINVAL, why.c_str());
    *valid = sketch_valid(sketch, sh, values) ? 1 : 0;
    return TUNER_OK;
}
