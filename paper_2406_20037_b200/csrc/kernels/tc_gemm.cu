// tc_gemm.cu — sketches TC_GEMM_BF16 and TC_IGEMM_CONV_BF16 on the 5th-generation
// tensor cores.
//   dense / bmm : Y[b,m,n] (fp32) = sum_k X[b,m,k] W[b,n,k],  X, W bf16
//   conv2d      : Y[n,p,q,k] (fp32) = sum_{r,s,c} X[n,p*sh-ph+r*dh,q*sw-pw+s*dw,c] W[k,r,s,c]
//
// The sketch (Def. 2.1): tile the output into BM x BN tiles (x SPLIT_K slices of
// the reduction); stage BK-wide reduction slices of A and B through a
// STAGES-deep shared-memory ring filled by TMA (128-byte swizzle, one mbarrier
// pair per stage); accumulate in TMEM with tcgen05.mma issued by one thread
// (kind::f16, fp32 accumulate); drain TMEM with tcgen05.ld in four epilogue
// warps straight to global memory, or with vector reductions
// (red.global.add.v4.f32) into a zeroed Y when SPLIT_K > 1.
//
// BM = 128: one CTA per tile, UMMA 128 x BN x 16 (cta_group::1).
// BM = 256: a CTA pair (cluster of 2 on one TPC) per tile, UMMA 256 x BN x 16
// (cta_group::2): each CTA stages 128 rows of A and BN/2 rows of B, the leader
// issues the MMA over both CTAs' shared memory, and each CTA's TMEM holds its
// 128 accumulator rows — half the B traffic per SM of two 1-CTA tiles.
//
// Persistent: one CTA (pair) per SM (pair) slot walks the work units
// (tile, k-slice) round-robin.  The TMEM accumulator is double-buffered
// (2 x BN columns), so the epilogue of unit i overlaps the MMAs of unit i+1 and
// the TMA ring never drains between units.
//
// Implicit GEMM (TQ > 0): a 128-row M sub-tile is a TP x TQ rectangle of output
// pixels of one image (TP = 128 / TQ).  For filter tap (r, s) and channel block
// c0 its A slice is ONE 4-D TMA box of X (NHWC) starting at
// (c0, q0*sw - pw + s*dw, p0*sh - ph + r*dh, n) with traversal strides (sw, sh):
// the hardware does the im2col gather, the conv stride, and the zero padding
// (out-of-bounds fill).  B is W (KRSC) as a 4-D box (c0, s, r, k0).
// Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
// Knobs: BM, BN, BK, STAGES, SPLIT_K, TILE_Q (conv only).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"

// the halo instantiations return from the producer / MMA segment loops before the generic k-block
// loops (if constexpr + continue): those are dead code there, by design
#pragma nv_diag_suppress 128

namespace db200 {


// STAGES is a runtime knob (the ring depth only sizes shared memory and indexes the ring).
// EW = epilogue warps: 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each draining every
// other 32-column chunk: twice the TMA stores in flight per SM)
template <int BN, int BK, int CG, int EW = 4>
struct TcCfg {
    static constexpr int BM = 128;  // rows of A per CTA
    static constexpr int BNC = BN / CG;  // rows of B per CTA
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BNC * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // double-buffered accumulator, allocated as a power of two >= 32 columns (BN = 192 -> 512)
    static constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
    // epilogue staging for TMA stores: per epilogue warp one 64-column TMEM chunk = two
    // 32-row x 32-column fp32 boxes whose 128-byte rows are stored 128B-swizzled (bank-conflict
    // free st.shared.v4, and the layout the tensor map's SWIZZLE_128B expects), written with ONE
    // proxy fence and two TMA stores per chunk; 1024-byte aligned, right after the stages
    // (EPI knob: 1 = the boxes go out as TMA stores; 2 = the warp reads its boxes back row-major
    // and writes them with coalesced 128-byte st.global / red.global segments -- no async proxy,
    // no TMA queue shared with the operand loads)
    static constexpr int EPI_BOX = 32 * 32;
    static constexpr int EPI_BYTES = 4 * 2 * EPI_BOX * 4;
    static_assert(EPI_BYTES == kTcEpiBytes, "epilogue staging size");
    static constexpr int MAX_STAGES = 8;
    static constexpr size_t smem(int stages) { return 1024 + (size_t)stages * STAGE_BYTES + (size_t)EPI_BYTES + 256; }
    static constexpr int THREADS = 64 + 32 * EW;
    static constexpr int CH = EW == 4 ? (BN < 64 ? BN : 64) : 32;  // columns per TMEM drain and staging
    static constexpr int CSTEP = CH * (EW / 4);                   // column stride between a warp's chunks
};

struct TcParams {
    int M, N, K;  // GEMM view (conv: M = N*P*Q, N = K_out, K = R*S*C)
    int kblocks, split;
    int m_tiles;                  // 128-row sub-tiles per batch (conv: images x pixel tiles)
    int mp_tiles, n_tiles, batch;  // tiles of the CTA group (CG sub-tiles each)
    int units;                    // SCHED 0: batch * mp_tiles * n_tiles * split
    int sched;                    // 0 = tiles (+ split-K), 1 = stream-K, 2 = full waves by tile + k-chunked rest
    int raster;                   // tile order: 0 = M fastest, 1 = N fastest
    int epi;                      // EPI knob: 1 = TMA-store epilogue, 2 = coalesced st.global epilogue
    int stages;                   // STAGES knob: depth of the TMA -> MMA shared-memory ring
    int dp_tiles;                 // SCHED 2: tiles handled whole (a multiple of the group count)
    int rem_tiles, rem_chunks;    // SCHED 2: remainder tiles and k-chunks per remainder tile
    long long total_iters;        // SCHED 1/2: streamed k-block iterations (tiles - dp_tiles) * kblocks
    unsigned* flags;              // SCHED 1: per workspace slot (group x CTA): 1 = partial parked
    float* ws;                    // SCHED 1: [slot][128][BN] partial accumulators of tails
    float* C;
    unsigned long long* trace;  // debug (DB200_TC_TRACE): [CTA][16] globaltimer stamps, else nullptr
    // implicit GEMM
    int P, Q, S, CB;  // CB = channel blocks of BK per tap
    int sh, sw, ph, pw, dh, dw;
    int tiles_p, tiles_q;
    // halo tiles (TILE_Q = 128): R input-row windows of 128 + S - 1 pixels per channel block,
    // each win_bytes apart (1024-aligned), a_stage_bytes = R * win_bytes per A-ring stage
    int R, win_bytes, a_stage_bytes;
    int N_img;       // conv: images (a sub-tile with image >= N_img is padding)
    int contiguous;  // SCHED 0 with contiguous unit ranges per group (halo: runs down the rows)
};

// epilogue modes of a segment: plain store; split-K reduction into a zeroed Y;
// stream-K head (wait for the tile's tails, add their partials, store); stream-K
// tail (park the partial in the group's workspace slot and signal)
enum : int { EPI_STORE = 0, EPI_RED = 1, EPI_HEAD = 2, EPI_TAIL = 3 };

struct Seg {
    int tile;                  // linear tile index (m fastest), SCHED 1 flag index base
    int bz, mt, nt, kb0, nkb;  // mt = index of the CTA group's tile
    int mode;
    int ntails;                // SCHED 1/2: segments of this tile after its head
    int tstride;               // groups between consecutive segments of a split tile (SCHED 1: 1)
};

// Walks the segments (tile, k range) of one CTA group.  SCHED 0: units u = g, g+G, ...
// (tile x split-K slice, balanced slices).  SCHED 1 (stream-K): the contiguous share
// [g*T/G, (g+1)*T/G) of all T = tiles * kblocks iterations, cut at tile boundaries.
struct SegIter {
    long long cur, end;
    int u;
    __device__ SegIter(const TcParams& p, int g, int G) {
        u = g;
        if (p.contiguous) {  // group g takes units [g U / G, (g+1) U / G) in order
            cur = (long long)g * p.units / G;
            end = (long long)(g + 1) * p.units / G;
        } else if (p.sched == 2) {  // the remainder unit of this group (if any): [g, g + 1)
            cur = g;
            end = g + 1;
        } else {
            cur = (long long)g * p.total_iters / G;
            end = (long long)(g + 1) * p.total_iters / G;
        }
    }
    __device__ bool next(const TcParams& p, int G, Seg& s) {
        int t;
        if (p.contiguous) {
            if (cur >= end) return false;
            t = (int)cur++;
            s.kb0 = 0;
            s.nkb = p.kblocks;
            s.mode = EPI_STORE;
            s.ntails = 0;
        } else if (p.sched == 0) {
            if (u >= p.units) return false;
            const int kz = u % p.split;
            t = u / p.split;
            s.kb0 = (int)((long long)kz * p.kblocks / p.split);  // non-empty when split <= kblocks
            s.nkb = (int)((long long)(kz + 1) * p.kblocks / p.split) - s.kb0;
            s.mode = p.split > 1 ? EPI_RED : EPI_STORE;
            u += G;
        } else if (u < p.dp_tiles) {  // SCHED 2: the full waves go tile by tile
            t = u;
            s.kb0 = 0;
            s.nkb = p.kblocks;
            s.mode = EPI_STORE;
            s.ntails = 0;
            u += G;
        } else if (p.sched == 2) {
            // SCHED 2 remainder: R = tiles - dp_tiles tiles, each cut into S equal k-chunks;
            // unit v = chunk * R + tile (chunk-major) goes to group v, so the groups working at
            // the same time share few k-slices (their operand reads overlap in L2); chunk 0
            // is the head, chunks 1..S-1 are tails parked by groups v + R, v + 2R, ...
            const int R = p.rem_tiles, S = p.rem_chunks, v = (int)cur;
            if (cur >= end || v >= R * S) return false;
            cur = end;  // one remainder unit per group
            const int c = v / R;
            t = p.dp_tiles + v % R;
            s.kb0 = (int)((long long)c * p.kblocks / S);
            s.nkb = (int)((long long)(c + 1) * p.kblocks / S) - s.kb0;
            s.mode = S == 1 ? EPI_STORE : (c == 0 ? EPI_HEAD : EPI_TAIL);
            s.ntails = c == 0 ? S - 1 : 0;
            s.tstride = R;
        } else {
            if (cur >= end) return false;
            const int tl = (int)(cur / p.kblocks);  // tile index within the streamed remainder
            t = p.dp_tiles + tl;
            s.kb0 = (int)(cur - (long long)tl * p.kblocks);
            const long long left = end - cur;
            s.nkb = (int)((long long)(p.kblocks - s.kb0) < left ? (p.kblocks - s.kb0) : left);
            const bool head = s.kb0 == 0, whole = head && s.nkb == p.kblocks;
            // a head that is not the whole tile is the LAST segment of its group's range and
            // a tail is the FIRST one: heads wait for tails finished early -- no chain
            s.mode = whole ? EPI_STORE : (head ? EPI_HEAD : EPI_TAIL);
            // groups sharing this tile: g(i) = ceil((i+1) G / T) - 1 owns iteration i
            const long long T = p.total_iters, i0 = (long long)tl * p.kblocks, i1 = i0 + p.kblocks - 1;
            s.ntails = (int)(((i1 + 1) * G + T - 1) / T - ((i0 + 1) * G + T - 1) / T);
            s.tstride = 1;
            cur += s.nkb;
        }
        s.tile = t;
        const int per = p.mp_tiles * p.n_tiles;
        s.bz = t / per;
        int r = t - s.bz * per;
        if (p.raster == 0) {  // m fastest: concurrent CTAs share the B (weight) panel in L2
            s.mt = r % p.mp_tiles;
            s.nt = r / p.mp_tiles;
        } else if (p.raster == 1) {  // n fastest: concurrent CTAs share the A panel
            s.nt = r % p.n_tiles;
            s.mt = r / p.n_tiles;
        } else if (p.raster == 2) {  // bands of 8 m-tiles, m fastest inside a band, then n
            const int band = r / (8 * p.n_tiles), rows = min(8, p.mp_tiles - band * 8);
            r -= band * 8 * p.n_tiles;
            s.mt = band * 8 + r % rows;
            s.nt = r / rows;
        } else {  // bands of 8 n-tiles, n fastest inside a band, then m
            const int band = r / (8 * p.mp_tiles), cols = min(8, p.n_tiles - band * 8);
            r -= band * 8 * p.mp_tiles;
            s.nt = band * 8 + r % cols;
            s.mt = r / cols;
        }
        return true;
    }
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// trace slots: 0 start, 1..4 epilogue segment j ready (acc_full), 5..8 segment j done,
// 9 head flags seen, 10 end; halo: 11 / 12 MMA at segment 1 / 2 (accumulator free), 13 segment 2
// windows landed, 14 producer issued segment 2 windows, 15 MMA issued segment 2
#define TC_TRACE(slot)                                                                   \
    do {                                                                                 \
        if (p.trace) p.trace[(size_t)blockIdx.x * 16 + (slot)] = gtimer();               \
    } while (0)

__device__ __forceinline__ void epi_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int BN, int BK, int TQ, int CG, int EW>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    tc_gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmY, const TcParams p) {
    using Cfg = TcCfg<BN, BK, CG, EW>;
    const int STAGES = p.stages;
    constexpr int BM = Cfg::BM;
    constexpr bool CONV = TQ > 0;
    constexpr bool HALO = TQ == 128;  // halo row tiles: A staged once per channel block, taps = shifted views
    constexpr int TP = CONV ? BM / TQ : 1;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // shared memory:
    //   generic: [STAGES x (A slice + B slice of one k-block)][epilogue staging][barriers]
    //   halo:    [NW = STAGES window slots of CB x (128 + S - 1) input pixels][B resident: all CB x R*S
    //             taps of the n-tile][epilogue staging][barriers]
    uint8_t* aring = base;
    uint8_t* ring = base + (HALO ? STAGES * p.a_stage_bytes : 0);
    const int ring_bytes = HALO ? p.CB * p.R * p.S * Cfg::B_BYTES : STAGES * Cfg::STAGE_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + ring_bytes + Cfg::EPI_BYTES);
    const int NB = HALO ? 1 : STAGES;  // halo: one full / empty pair guards the resident B
    uint64_t* full = bars;
    uint64_t* empty = bars + NB;
    uint64_t* acc_full = bars + 2 * NB;       // [2] MMA -> epilogue
    uint64_t* acc_empty = bars + 2 * NB + 2;  // [2] epilogue -> MMA
    uint64_t* full_w = bars + 2 * NB + 4;     // halo: [NW] window slot loaded (TMA -> MMA)
    uint64_t* empty_w = full_w + (HALO ? STAGES : 0);  // halo: [NW] window slot released (MMA -> TMA)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty_w + (HALO ? STAGES : 0));
    float* epi_smem = reinterpret_cast<float*>(ring + ring_bytes);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? tc::cluster_ctarank() : 0u;
    if (threadIdx.x == 0) TC_TRACE(0);
    // programmatic dependent launch: the next kernel in the stream may be launched now (its CTAs
    // become resident as this kernel's exit); this kernel's own TMA loads and stores wait for its
    // predecessor (griddepcontrol.wait) -- only the prologue (barriers, TMEM, tensor maps) overlaps
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int group = blockIdx.x / CG, ngroups = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < NB; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), CG);  // leader: own arrive.expect_tx (+ the peer's arrive)
            tc::mbar_init(tc::smem_u32(&empty[s]), 1);
        }
        if constexpr (HALO) {
            for (int s = 0; s < STAGES; ++s) {
                tc::mbar_init(tc::smem_u32(&full_w[s]), CG);
                tc::mbar_init(tc::smem_u32(&empty_w[s]), 1);
            }
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(tc::smem_u32(&acc_full[a]), 1);
            tc::mbar_init(tc::smem_u32(&acc_empty[a]), EW * CG);  // one arrive per epilogue warp of the group
        }
        tc::fence_barrier_init();
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
    }
    if (warp == 1) {
        if constexpr (CG == 2) tc::tmem_alloc_cg2<Cfg::TMEM_COLS>(tc::smem_u32(tmem_slot));
        else tc::tmem_alloc<Cfg::TMEM_COLS>(tc::smem_u32(tmem_slot));
    }
    tc::tc_fence_before();
    if constexpr (CG == 2) tc::cluster_sync();
    else __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // this CTA's 128-row sub-tile of the group's tile
    auto sub_tile = [&](const Seg& w) { return w.mt * CG + (int)rank; };
    // conv: (image, first output row, first output column) of this CTA's 128-pixel sub-tile;
    // image >= N marks a padding sub-tile (TMA zero-fills its loads, its stores are clipped).
    // Halo tiles run down the output rows (p fastest, then the column tile, then the image) so a
    // CTA's consecutive tiles share R-1 input rows; a CTA pair splits the rows into two halves.
    struct Px {
        int img, p0, q0;
    };
    auto px_of = [&](const Seg& w) {
        Px x;
        if constexpr (HALO) {
            const int ph = (p.P + CG - 1) / CG;
            const int t = w.mt / ph;
            x.p0 = w.mt % ph + (int)rank * ph;
            x.q0 = (t % p.tiles_q) * 128;
            x.img = t / p.tiles_q;
            if (x.p0 >= p.P) x.img = p.N_img;  // the pair's second half ran past the last row
        } else {
            const int mt = sub_tile(w);
            x.q0 = (mt % p.tiles_q) * TQ;
            const int t = mt / p.tiles_q;
            x.p0 = (t % p.tiles_p) * TP;
            x.img = t / p.tiles_p;
        }
        return x;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: one continuous ring across units
            // X / W may be written by the preceding kernel; behind a split-K zeroing kernel (plainly
            // serialised) every earlier kernel is already complete
            if (p.split == 1) griddep_wait();
            int ps = 0;         // ring stage of the next k-block
            uint32_t pph = 0;   // and its phase parity
            int b_nt = -1, b_loads = 0, wseq = 0, r_mt = -2, r_row = 0, r_nt = -1;  // halo state
            const int ph_rows_p = (p.P + CG - 1) / CG;
            int pseg = 0;
            SegIter si(p, group, ngroups);
            Seg w;
            while (si.next(p, ngroups, w)) {
                const int mt = sub_tile(w);
                int img = w.bz, p0 = 0, q0 = 0;
                if constexpr (CONV) {
                    const Px x = px_of(w);
                    img = x.img;
                    p0 = x.p0;
                    q0 = x.q0;
                }
                const int nb = w.nt * BN + (int)rank * Cfg::BNC;
                if constexpr (HALO) {
                    const int RS = p.R * p.S, NW = STAGES;
                    // B resident: every (channel block, tap) slice of the n-tile, loaded when it changes
                    if (w.nt != b_nt) {
                        tc::mbar_wait(tc::smem_u32(&empty[0]), ((uint32_t)b_loads & 1u) ^ 1u);
                        const uint32_t fb = tc::smem_u32(&full[0]);
                        if (rank == 0) tc::mbar_expect_tx(fb, (uint32_t)(CG * p.CB * RS * Cfg::B_BYTES));
                        else tc::mbar_arrive_remote(fb, 0);
                        for (int cb = 0; cb < p.CB; ++cb)
                            for (int tap = 0; tap < RS; ++tap) {
                                const uint32_t sb = tc::smem_u32(ring + (cb * RS + tap) * Cfg::B_BYTES);
                                const int fr = tap / p.S, fs = tap - fr * p.S;
                                if constexpr (CG == 2) tc::tma_load_4d_cg2(sb, &tmB, fb, cb * 64, fs, fr, nb);
                                else tc::tma_load_4d(sb, &tmB, fb, cb * 64, fs, fr, nb);
                            }
                        b_nt = w.nt;
                        ++b_loads;
                    }
                    // input-row windows (one TMA box of 128 + S - 1 pixels per channel block, OOB =
                    // padding): all R for the first tile of a run, then the one new row per tile.  The
                    // run rule is the MMA issuer's, on the group's tile index (both CTAs of a pair and
                    // the issuer must agree; a pair's padding row past P continues its run)
                    const bool cont = w.mt == r_mt + 1 && r_row + 1 < ph_rows_p && w.nt == r_nt;
                    r_row = cont ? r_row + 1 : w.mt % ph_rows_p;
                    r_mt = w.mt;
                    const uint32_t wb = (uint32_t)(p.CB * (128 + p.S - 1) * 128);
                    for (int r = cont ? p.R - 1 : 0; r < p.R; ++r, ++wseq) {
                        const int slot = wseq % NW;
                        tc::mbar_wait(tc::smem_u32(&empty_w[slot]), ((uint32_t)(wseq / NW) & 1u) ^ 1u);
                        const uint32_t fa = tc::smem_u32(&full_w[slot]);
                        if (rank == 0) tc::mbar_expect_tx(fa, CG * wb);
                        else tc::mbar_arrive_remote(fa, 0);
                        const uint32_t wa = tc::smem_u32(aring + slot * p.a_stage_bytes);
                        for (int cb = 0; cb < p.CB; ++cb) {
                            const uint32_t dst = wa + (uint32_t)(cb * p.win_bytes);
                            if constexpr (CG == 2)
                                tc::tma_load_4d_cg2(dst, &tmA, fa, cb * 64, q0 - p.pw, p0 - p.ph + r, img);
                            else tc::tma_load_4d(dst, &tmA, fa, cb * 64, q0 - p.pw, p0 - p.ph + r, img);
                        }
                    }
                    r_nt = w.nt;
                    if (pseg == 2) TC_TRACE(14);  // producer: windows of segment 2 issued
                    ++pseg;
                    continue;
                }
                // (channel block, filter column, filter row) of the segment's first k-block, then
                // carried: no integer division per k-block
                int cb = 0, fs = 0, fr = 0;
                if constexpr (CONV) {
                    cb = w.kb0 % p.CB;
                    const int rs = w.kb0 / p.CB;
                    fs = rs % p.S;
                    fr = rs / p.S;
                }
                for (int i = 0; i < w.nkb; ++i) {
                    const int s = ps;
                    const uint32_t ph = pph;
                    if (++ps == STAGES) {
                        ps = 0;
                        pph ^= 1u;
                    }
                    tc::mbar_wait(tc::smem_u32(&empty[s]), ph ^ 1u);
                    const uint32_t fb = tc::smem_u32(&full[s]);
                    if (rank == 0) tc::mbar_expect_tx(fb, CG * Cfg::STAGE_BYTES);
                    else tc::mbar_arrive_remote(fb, 0);
                    const uint32_t sa = tc::smem_u32(ring + s * Cfg::STAGE_BYTES);
                    const uint32_t sb = sa + Cfg::A_BYTES;
                    const int kb = w.kb0 + i;
                    if constexpr (CONV) {
                        const int wq = q0 * p.sw - p.pw + fs * p.dw;
                        const int hp = p0 * p.sh - p.ph + fr * p.dh;
#pragma unroll
                        for (int a = 0; a < BK / 64; ++a) {
                            const int c0 = cb * BK + a * 64;
                            if constexpr (CG == 2) {
                                tc::tma_load_4d_cg2(sa + a * BM * 128, &tmA, fb, c0, wq, hp, img);
                                tc::tma_load_4d_cg2(sb + a * Cfg::BNC * 128, &tmB, fb, c0, fs, fr, nb);
                            } else {
                                tc::tma_load_4d(sa + a * BM * 128, &tmA, fb, c0, wq, hp, img);
                                tc::tma_load_4d(sb + a * Cfg::BNC * 128, &tmB, fb, c0, fs, fr, nb);
                            }
                        }
                        if (++cb == p.CB) {
                            cb = 0;
                            if (++fs == p.S) {
                                fs = 0;
                                ++fr;
                            }
                        }
                    } else {
                        const int k0 = kb * BK;
#pragma unroll
                        for (int a = 0; a < BK / 64; ++a) {
                            if constexpr (CG == 2) {
                                tc::tma_load_3d_cg2(sa + a * BM * 128, &tmA, fb, k0 + a * 64, mt * BM, w.bz);
                                tc::tma_load_3d_cg2(sb + a * Cfg::BNC * 128, &tmB, fb, k0 + a * 64, nb, w.bz);
                            } else {
                                tc::tma_load_3d(sa + a * BM * 128, &tmA, fb, k0 + a * 64, mt * BM, w.bz);
                                tc::tma_load_3d(sb + a * Cfg::BNC * 128, &tmB, fb, k0 + a * 64, nb, w.bz);
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ---- MMA issuer (the leader CTA of a pair): the whole warp, one elected lane issues
            constexpr uint32_t idesc = tc::idesc_bf16(BM * CG, BN);
            int j = 0;
            int ms = 0;        // ring stage of the next k-block (generic)
            uint32_t mph = 0;  // and its phase parity
            const uint32_t ring_u32 = tc::smem_u32(ring);
            // halo state: the resident B's n-tile and load count; the window slot of input row 0 of
            // the current tile (s0) and the slot / phase the next fresh window lands in
            int b_nt = -1, b_loads = 0, s0 = 0, nslot = 0, prev_mt = -2, row = 0;
            uint32_t nph = 0;
            bool have_run = false;
            const int ph_rows = (p.P + CG - 1) / CG;
            SegIter si(p, group, ngroups);
            Seg w;
            for (; si.next(p, ngroups, w); ++j) {
                const int a = j & 1;
                tc::mbar_wait(tc::smem_u32(&acc_empty[a]), ((uint32_t)(j >> 1) & 1u) ^ 1u);
                tc::tc_fence_after();
                const uint32_t acc = tmem + (uint32_t)(a * BN);
                if constexpr (HALO) {
                    const int NW = STAGES;
                    auto commit = [&](uint32_t bar) {
                        if constexpr (CG == 2) tc::umma_commit_cg2_w(bar);
                        else tc::umma_commit_w(bar);
                    };
                    if (w.nt != b_nt) {  // a new resident B: release the old one once its MMAs finish
                        if (b_loads > 0) commit(tc::smem_u32(&empty[0]));
                        tc::mbar_wait(tc::smem_u32(&full[0]), (uint32_t)b_loads & 1u);
                        tc::tc_fence_after();
                        b_nt = w.nt;
                        ++b_loads;
                        prev_mt = -2;  // windows do not carry across n-tiles
                    }
                    // the next output row of the same run shares R-1 input rows with this one
                    const bool cont = w.mt == prev_mt + 1 && row + 1 < ph_rows;
                    row = cont ? row + 1 : w.mt % ph_rows;
                    prev_mt = w.mt;
                    // release the windows this tile drops (their readers are all issued: the commit
                    // arrives when they complete), then wait for the rows it adds
                    int fresh;
                    if (cont) {
                        commit(tc::smem_u32(&empty_w[s0]));
                        s0 = s0 + 1 == NW ? 0 : s0 + 1;
                        fresh = p.R - 1;
                    } else {
                        if (have_run) {
                            int sl = s0;
                            for (int r = 0; r < p.R; ++r) {
                                commit(tc::smem_u32(&empty_w[sl]));
                                sl = sl + 1 == NW ? 0 : sl + 1;
                            }
                        }
                        s0 = nslot;
                        fresh = 0;
                        have_run = true;
                    }
                    if (lane == 0 && (j == 1 || j == 2)) TC_TRACE(10 + j);  // MMA: accumulator free, before the window waits
                    for (int r = fresh; r < p.R; ++r) {
                        tc::mbar_wait(tc::smem_u32(&full_w[nslot]), nph);
                        if (++nslot == NW) {
                            nslot = 0;
                            nph ^= 1u;
                        }
                    }
                    tc::tc_fence_after();
                    if (lane == 0 && j == 2) TC_TRACE(13);  // MMA: windows of segment 2 landed
                    // tap (r, s) of channel block cb = rows s .. s+127 of window r: a whole-row shift of
                    // the start address (the 128B swizzle is a function of the absolute address, so the
                    // view stays consistent with the TMA-written layout; tools/umma_shift_probe.cu).
                    // Descriptors advance by constants: B slices are stored in (cb, r, s) order.
                    uint64_t db = tc::sdesc_sw128(ring_u32);
                    const uint64_t da_ring = tc::sdesc_sw128(tc::smem_u32(aring));
                    const uint32_t slot_step = (uint32_t)p.a_stage_bytes >> 4, win_step = (uint32_t)p.win_bytes >> 4;
                    uint32_t accum = 0u;
                    for (int cb = 0; cb < p.CB; ++cb) {
                        int sl = s0;
                        for (int fr = 0; fr < p.R; ++fr) {
                            const uint64_t drow = da_ring + (uint64_t)(sl * slot_step + cb * win_step);
                            sl = sl + 1 == NW ? 0 : sl + 1;
                            for (int fs = 0; fs < p.S; ++fs) {
                                const uint64_t da = drow + (uint64_t)(fs * 8);  // fs rows of 128 B
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    if constexpr (CG == 2) tc::umma_bf16_cg2_w(acc, da + 2 * k, db + 2 * k, idesc, accum);
                                    else tc::umma_bf16_w(acc, da + 2 * k, db + 2 * k, idesc, accum);
                                    accum = 1u;
                                }
                                db += (uint64_t)(Cfg::B_BYTES >> 4);
                            }
                        }
                    }
                    commit(tc::smem_u32(&acc_full[a]));
                    if (lane == 0 && j == 2) TC_TRACE(15);  // MMA: segment 2 issued
                    continue;
                }
                // the issue loop is one thread's dependent scalar code: ring index and phase are
                // carried (no division by the runtime STAGES), descriptors are a per-stage base plus
                // compile-time offsets (the 14-bit address field of a descriptor is addr >> 4)
                for (int i = 0; i < w.nkb; ++i) {
                    const int s = ms;
                    const uint32_t ph = mph;
                    if (++ms == STAGES) {
                        ms = 0;
                        mph ^= 1u;
                    }
                    tc::mbar_wait(tc::smem_u32(&full[s]), ph);
                    tc::tc_fence_after();
                    const uint32_t sa = ring_u32 + (uint32_t)(s * Cfg::STAGE_BYTES);
                    const uint64_t da0 = tc::sdesc_sw128(sa), db0 = tc::sdesc_sw128(sa + Cfg::A_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint32_t offa = ((k / 4) * BM * 128 + (k % 4) * 32) >> 4;
                        const uint32_t offb = ((k / 4) * Cfg::BNC * 128 + (k % 4) * 32) >> 4;
                        if constexpr (CG == 2) tc::umma_bf16_cg2_w(acc, da0 + offa, db0 + offb, idesc, (i > 0 || k > 0) ? 1u : 0u);
                        else tc::umma_bf16_w(acc, da0 + offa, db0 + offb, idesc, (i > 0 || k > 0) ? 1u : 0u);
                    }
                    // frees the stage (in both CTAs of a pair) when these MMAs finish
                    if constexpr (CG == 2) tc::umma_commit_cg2_w(tc::smem_u32(&empty[s]));
                    else tc::umma_commit_w(tc::smem_u32(&empty[s]));
                }
                if constexpr (CG == 2) tc::umma_commit_cg2_w(tc::smem_u32(&acc_full[a]));
                else tc::umma_commit_w(tc::smem_u32(&acc_full[a]));
            }
        }
    } else {  // ---- epilogue: TMEM -> registers -> global
        griddep_wait();  // Y is written by the preceding kernel (split-K: zeroed by it)
        const int q = warp & 3;          // TMEM lane quadrant this warp may access (warp % 4)
        const int ew = warp - 2;         // epilogue warp index 0..EW-1
        const int half = ew >> 2;        // EW = 8: which of the quadrant's two warps (chunk parity)
        const int trow = q * 32 + lane;  // row of the 128-row sub-tile held by this thread
        const bool vec_ok = (p.N % 4) == 0;  // TMA needs 16-byte global strides
        int j = 0;
        SegIter si(p, group, ngroups);
        Seg w;
        for (; si.next(p, ngroups, w); ++j) {
            const int mt = sub_tile(w);
            const int a = j & 1;
            bool row_ok = mt < p.m_tiles;
            long long orow;  // output row index (GEMM row or NPQ pixel)
            Px px{0, 0, 0};
            if constexpr (CONV) {
                px = px_of(w);
                const int pp = px.p0 + trow / TQ, qq = px.q0 + trow % TQ;
                row_ok = px.img < p.N_img && pp < p.P && qq < p.Q;
                orow = ((long long)px.img * p.P + pp) * p.Q + qq;
            } else {
                const int m = mt * BM + trow;
                row_ok = row_ok && m < p.M;
                orow = (long long)w.bz * p.M + m;
            }
            // TMA-store box origin of this warp's 32 rows: dense (col, row, batch); conv
            // (k, q, p, image) with the rows forming a (32 / TQ) x TQ pixel rectangle
            int bx1 = 0, bx2 = 0, bx3 = 0;
            if constexpr (CONV) {
                constexpr int TQW = TQ < 32 ? TQ : 32;
                bx1 = px.q0 + ((q * 32) % TQ);
                bx2 = px.p0 + (q * 32) / TQ * (TQ / TQW);
                bx3 = px.img;
            } else {
                bx1 = mt * BM + q * 32;
                bx2 = w.bz;
            }
            tc::mbar_wait(tc::smem_u32(&acc_full[a]), (uint32_t)(j >> 1) & 1u);
            tc::tc_fence_after();
            if (warp == 2 && lane == 0 && j < 4) TC_TRACE(1 + j);
            const int slot = group * CG + (int)rank;  // this group's workspace slot (stream-K)
            if (w.mode == EPI_HEAD) {  // wait until every tail of this tile parked its partial
                if (warp == 2 && lane == 0) {
                    for (int tl = 1; tl <= w.ntails; ++tl) {
                        const unsigned* f = p.flags + (slot + tl * w.tstride * CG);
                        unsigned v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                        } while (v == 0u);
                    }
                    TC_TRACE(9);
                }
                epi_bar(1, 32 * EW);
            }
            const bool red = w.mode == EPI_RED;
            // a parked partial is stored thread-major, [BN/16][128 rows][16], so each warp
            // writes (and its head later reads) 2 KB contiguous per 16-column group
            float* crow = w.mode == EPI_TAIL ? p.ws + (long long)slot * 128 * 256 + trow * 16
                                             : p.C + orow * p.N;
            const int n0 = w.mode == EPI_TAIL ? 0 : w.nt * BN;
            const bool live = w.mode == EPI_TAIL ? true : row_ok;
            const int ncols = w.mode == EPI_TAIL ? BN : p.N;
            constexpr int CH = Cfg::CH;  // columns per TMEM drain: several loads, one wait
#pragma unroll 1
            for (int c0 = half * CH; c0 < BN; c0 += Cfg::CSTEP) {
                uint32_t r[CH / 16][16];
#pragma unroll
                for (int g = 0; g < CH / 16; ++g)
                    tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * BN + c0 + g * 16), r[g]);
                tc::tmem_ld_wait();
                if (w.mode == EPI_HEAD && live) {
                    // add the tails' parked partials (same rows, same columns): all of a tail's
                    // loads for this chunk are issued before any add, so they overlap in flight
                    for (int tl = 1; tl <= w.ntails; ++tl) {
                        const float4* pp = reinterpret_cast<const float4*>(
                            p.ws + (long long)(slot + tl * w.tstride * CG) * 128 * 256 +
                            (long long)(c0 / 16) * (128 * 16) + trow * 16);
                        float4 x[CH / 16][4];
#pragma unroll
                        for (int g = 0; g < CH / 16; ++g)
#pragma unroll
                            for (int v = 0; v < 4; ++v) x[g][v] = __ldcg(pp + g * (128 * 16 / 4) + v);
#pragma unroll
                        for (int g = 0; g < CH / 16; ++g)
#pragma unroll
                            for (int v = 0; v < 4; ++v) {
                                r[g][4 * v] = __float_as_uint(__uint_as_float(r[g][4 * v]) + x[g][v].x);
                                r[g][4 * v + 1] = __float_as_uint(__uint_as_float(r[g][4 * v + 1]) + x[g][v].y);
                                r[g][4 * v + 2] = __float_as_uint(__uint_as_float(r[g][4 * v + 2]) + x[g][v].z);
                                r[g][4 * v + 3] = __float_as_uint(__uint_as_float(r[g][4 * v + 3]) + x[g][v].w);
                            }
                    }
                }
                if (w.mode != EPI_TAIL && vec_ok) {
                    // staged through shared memory: the chunk's CH/32 boxes of 32 rows x 32
                    // columns, lane = box row, 16-byte chunk c of a row at physical chunk
                    // c ^ (row & 7) (SWIZZLE_128B: conflict-free st.shared.v4 / ld.shared.v4)
                    static_assert(CH % 32 == 0, "staged chunks are 32 columns wide");
                    const uint32_t eb = tc::smem_u32(epi_smem + ew * (CH / 32) * Cfg::EPI_BOX);
                    if (p.epi == 1) {
                        if (lane == 0) tc::bulk_wait_read<0>();  // the previous chunk's stores have read it
                        __syncwarp();
                    }
#pragma unroll
                    for (int g = 0; g < CH / 16; ++g) {
                        const uint32_t brow = eb + (uint32_t)((g >> 1) * Cfg::EPI_BOX * 4 + lane * 128);
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const int c = (g & 1) * 4 + v;
                            tc::st_shared_v4(brow + (uint32_t)((c ^ (lane & 7)) << 4), r[g][4 * v], r[g][4 * v + 1],
                                             r[g][4 * v + 2], r[g][4 * v + 3]);
                        }
                    }
                    if (p.epi == 1) {  // TMA stores (OOB rows / columns / pixels are clipped by the map)
                        tc::fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
#pragma unroll
                            for (int b = 0; b < CH / 32; ++b) {
                                const uint32_t src = eb + (uint32_t)(b * Cfg::EPI_BOX * 4);
                                const int n = n0 + c0 + b * 32;
                                if constexpr (CONV) {
                                    if (red) tc::tma_red_add_4d(&tmY, src, n, bx1, bx2, bx3);
                                    else tc::tma_store_4d(&tmY, src, n, bx1, bx2, bx3);
                                } else {
                                    if (red) tc::tma_red_add_3d(&tmY, src, n, bx1, bx2);
                                    else tc::tma_store_3d(&tmY, src, n, bx1, bx2);
                                }
                            }
                            tc::bulk_commit();
                        }
                        continue;
                    }
                    // EPI 2: read the boxes back row-major, 8 lanes per 128-byte row segment, 4 rows
                    // per instruction, and write coalesced segments (rows / columns past the edge
                    // skipped; a row's global base comes from the lane that owns the row)
                    __syncwarp();
                    const int sub = lane >> 3, c = lane & 7;
#pragma unroll
                    for (int b = 0; b < CH / 32; ++b) {
                        const int n = n0 + c0 + b * 32 + 4 * c;
#pragma unroll 4
                        for (int it = 0; it < 8; ++it) {
                            const int rr = it * 4 + sub;
                            const float* rbase = reinterpret_cast<const float*>(
                                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(crow), rr));
                            const bool rok = __shfl_sync(0xffffffffu, live ? 1 : 0, rr) != 0;
                            uint32_t v0, v1, v2, v3;
                            tc::ld_shared_v4(eb + (uint32_t)(b * Cfg::EPI_BOX * 4 + rr * 128 + ((c ^ (rr & 7)) << 4)),
                                             v0, v1, v2, v3);
                            if (!rok || n >= ncols) continue;
                            float* dst = const_cast<float*>(rbase) + n;
                            if (red) tc::red_add_v4(dst, __uint_as_float(v0), __uint_as_float(v1), __uint_as_float(v2),
                                                    __uint_as_float(v3));
                            else *reinterpret_cast<uint4*>(dst) = make_uint4(v0, v1, v2, v3);
                        }
                    }
                    __syncwarp();  // every lane has read the boxes before the next chunk restages them
                    continue;
                }
#pragma unroll
                for (int g = 0; g < CH / 16; ++g) {
                    const int n = n0 + c0 + g * 16;
                    if (!live || n >= ncols) continue;
                    if ((vec_ok || w.mode == EPI_TAIL) && n + 16 <= ncols) {
                        float* dst = w.mode == EPI_TAIL ? crow + (long long)(n / 16) * (128 * 16) : crow + n;
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            float4 f = make_float4(__uint_as_float(r[g][4 * v]), __uint_as_float(r[g][4 * v + 1]),
                                                   __uint_as_float(r[g][4 * v + 2]), __uint_as_float(r[g][4 * v + 3]));
                            if (red) tc::red_add_v4(dst + 4 * v, f.x, f.y, f.z, f.w);
                            else *reinterpret_cast<float4*>(dst + 4 * v) = f;
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            if (n + jj < ncols) {
                                if (red) atomicAdd(crow + n + jj, __uint_as_float(r[g][jj]));
                                else crow[n + jj] = __uint_as_float(r[g][jj]);
                            }
                        }
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {  // this warp's accumulator lanes are drained
                if constexpr (CG == 2) tc::mbar_arrive_remote(tc::smem_u32(&acc_empty[a]), 0);
                else tc::mbar_arrive(tc::smem_u32(&acc_empty[a]));
            }
            if (warp == 2 && lane == 0 && j < 4) TC_TRACE(5 + j);
            if (w.mode == EPI_TAIL) {  // publish the parked partial (flag = 1)
                epi_bar(2, 32 * EW);
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.flags + slot), "r"(1u) : "memory");
                }
            } else if (w.mode == EPI_HEAD) {  // partials consumed: re-arm the tails' flags (0)
                epi_bar(2, 32 * EW);
                if (warp == 2 && lane == 0) {
                    for (int tl = 1; tl <= w.ntails; ++tl) p.flags[slot + tl * w.tstride * CG] = 0u;
                }
            }
        }
        if (lane == 0) tc::bulk_wait_all();  // this warp's TMA stores are complete
        __syncwarp();
    }
    tc::tc_fence_before();
    if constexpr (CG == 2) tc::cluster_sync();
    else __syncthreads();
    if (threadIdx.x == 0) TC_TRACE(10);
    if (warp == 1) {
        tc::tc_fence_after();
        if constexpr (CG == 2) tc::tmem_dealloc_cg2<Cfg::TMEM_COLS>(tmem);
        else tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
    }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)f;
    }
    return fn;
}

static bool encode(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box, const cuuint32_t* es) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// fp32 tensor (the output Y): 32-float (128-byte) box rows, 128B-swizzled in shared memory
static bool encode_f32(CUtensorMap* m, void* ptr, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                       const cuuint32_t* box, const cuuint32_t* es) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, ptr, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Co-resident CTA groups of an instantiation on the current device (computed once per device):
// cudaOccupancyMaxActiveClusters with the launch's block, dynamic shared memory and cluster
// shape (it accounts for the ~240 registers per thread of these kernels), capped by TMEM
// (512 columns per SM) and by the shared-memory bound; never more than one group per CG SMs
// times that.
// dynamic shared memory of a launch.  Halo (TQ = 128): STAGES window slots of a_stage bytes (one
// input row, every channel block) + the resident B (b_res bytes) instead of the k-block ring.
template <int BN, int BK, int TQ, int CG, int EW>
static size_t tc_smem_bytes(int stages, int a_stage, int b_res) {
    using Cfg = TcCfg<BN, BK, CG, EW>;
    if constexpr (TQ == 128)
        return 1024 + (size_t)stages * a_stage + (size_t)b_res + (size_t)Cfg::EPI_BYTES + 256;
    else return Cfg::smem(stages);
}

template <int BN, int BK, int TQ, int CG, int EW>
static long long tc_resident_groups(int num_sms, int stages, int a_stage, int b_res) {
    using Cfg = TcCfg<BN, BK, CG, EW>;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, long long> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    const auto key = std::make_tuple(dev, stages, a_stage, b_res);
    {
        std::lock_guard<std::mutex> g(mu);
        auto f = cache.find(key);
        if (f != cache.end()) return f->second;
    }
    const size_t smem = tc_smem_bytes<BN, BK, TQ, CG, EW>(stages, a_stage, b_res);
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(CG);
    cfg.blockDim = dim3(Cfg::THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, tc_gemm_bf16_kernel<BN, BK, TQ, CG, EW>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        clusters = 0;
    }
    int per_sm = (int)((228 * 1024) / (smem + 1024));
    const int tmem_per_sm = (int)(512 / Cfg::TMEM_COLS);
    per_sm = per_sm < tmem_per_sm ? per_sm : tmem_per_sm;
    per_sm = per_sm < 1 ? 1 : per_sm;
    long long g = (long long)(num_sms / CG) * per_sm;
    if (clusters > 0 && clusters < g) g = clusters;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = g;
    return g;
}

// 3-D K-major operand [batch][rows][K] -> box {64, box_rows, 1}
static bool make_kmajor_map(CUtensorMap* m, const void* ptr, int64_t batch, int64_t rows, int64_t K, int box_rows) {
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)(rows * K * 2)};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return encode(m, ptr, 3, dims, strides, box, es);
}

template <int BN, int BK, int TQ, int CG, int EW>
cudaError_t tc_launch(const LaunchCtx& c) {
    using Cfg = TcCfg<BN, BK, CG, EW>;
    constexpr bool CONV = TQ > 0;
    auto kern = tc_gemm_bf16_kernel<BN, BK, TQ, CG, EW>;
    static std::atomic<unsigned long long> optin{0};
    {
        cudaError_t e = smem_optin(optin, kern, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const ShapeInfo& s = *c.sh;
    CUtensorMap ta, tb;
    TcParams p;
    std::memset(&p, 0, sizeof(p));
    p.M = (int)s.M; p.N = (int)s.N; p.K = (int)s.K;
    p.split = c.split;
    p.C = (float*)c.y;
    p.n_tiles = (int)((s.N + BN - 1) / BN);
    if constexpr (CONV) {
        constexpr int TP = 128 / TQ;
        // X: NHWC as {C, W, H, N}, traversal strides (1, sw, sh, 1); box {64, TQ*sw, TP*sh, 1}
        // (halo, TQ = 128: one input-row window {64, 128 + S - 1, 1, 1}, stride 1)
        cuuint64_t xd[4] = {(cuuint64_t)s.c, (cuuint64_t)s.w, (cuuint64_t)s.h, (cuuint64_t)s.n};
        cuuint64_t xs[3] = {(cuuint64_t)s.c * 2, (cuuint64_t)(s.w * s.c * 2), (cuuint64_t)(s.h * s.w * s.c * 2)};
        cuuint32_t xb[4] = {64, (cuuint32_t)(TQ * s.sw), (cuuint32_t)(TP * s.sh), 1};
        cuuint32_t xe[4] = {1, (cuuint32_t)s.sw, (cuuint32_t)s.sh, 1};
        if constexpr (TQ == 128) {
            if (s.sh != 1 || s.sw != 1 || s.dh != 1 || s.dw != 1 || s.c % 64 || 128 + s.s - 1 > 256)
                return cudaErrorInvalidConfiguration;
            xb[1] = (cuuint32_t)(128 + s.s - 1);
            xb[2] = 1;
            if (c.sched != 0 || c.split != 1 || c.raster != 0 || c.stages < s.r + 1) return cudaErrorInvalidConfiguration;
            p.R = (int)s.r;
            p.win_bytes = (int)(((128 + s.s - 1) * 128 + 1023) / 1024 * 1024);  // one channel block's window
            p.a_stage_bytes = (int)(s.c / 64) * p.win_bytes;                       // a slot: one input row
            p.contiguous = 1;
        }
        // W: KRSC as {C, S, R, K}; box {64, 1, 1, BN / CG}
        cuuint64_t wd[4] = {(cuuint64_t)s.c, (cuuint64_t)s.s, (cuuint64_t)s.r, (cuuint64_t)s.k};
        cuuint64_t ws[3] = {(cuuint64_t)s.c * 2, (cuuint64_t)(s.s * s.c * 2), (cuuint64_t)(s.r * s.s * s.c * 2)};
        cuuint32_t wb[4] = {64, 1, 1, (cuuint32_t)Cfg::BNC};
        cuuint32_t we[4] = {1, 1, 1, 1};
        if (!encode(&ta, c.x, 4, xd, xs, xb, xe) || !encode(&tb, c.w, 4, wd, ws, wb, we))
            return cudaErrorInvalidValue;
        p.P = (int)s.p; p.Q = (int)s.q; p.S = (int)s.s;
        p.CB = (int)((s.c + BK - 1) / BK);
        p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
        p.tiles_q = (int)((s.q + TQ - 1) / TQ);
        p.tiles_p = (int)((s.p + TP - 1) / TP);
        p.kblocks = TQ == 128 ? p.CB : (int)(s.r * s.s) * p.CB;  // halo: a k-block = a channel block, all taps
        p.m_tiles = (int)s.n * p.tiles_p * p.tiles_q;
        p.N_img = (int)s.n;
        p.batch = 1;
    } else {
        if (!make_kmajor_map(&ta, c.x, s.batch, s.M, s.K, Cfg::BM) ||
            !make_kmajor_map(&tb, c.w, s.batch, s.N, s.K, Cfg::BNC))
            return cudaErrorInvalidValue;
        p.kblocks = (int)((s.K + BK - 1) / BK);
        p.m_tiles = (int)((s.M + Cfg::BM - 1) / Cfg::BM);
        p.batch = (int)s.batch;
    }
    // Y (fp32) for the TMA-store epilogue: one box = one epilogue warp's 32 rows x 32 columns
    CUtensorMap ty;
    std::memset(&ty, 0, sizeof(ty));
    if (s.N % 4 == 0) {
        bool ok;
        if constexpr (CONV) {
            constexpr int TQW = TQ < 32 ? TQ : 32;
            cuuint64_t yd[4] = {(cuuint64_t)s.k, (cuuint64_t)s.q, (cuuint64_t)s.p, (cuuint64_t)s.n};
            cuuint64_t ys[3] = {(cuuint64_t)s.k * 4, (cuuint64_t)(s.q * s.k * 4), (cuuint64_t)(s.p * s.q * s.k * 4)};
            cuuint32_t yb[4] = {32, (cuuint32_t)TQW, (cuuint32_t)(32 / TQW), 1};
            cuuint32_t ye[4] = {1, 1, 1, 1};
            ok = encode_f32(&ty, c.y, 4, yd, ys, yb, ye);
        } else {
            cuuint64_t yd[3] = {(cuuint64_t)s.N, (cuuint64_t)s.M, (cuuint64_t)s.batch};
            cuuint64_t ys[2] = {(cuuint64_t)s.N * 4, (cuuint64_t)(s.M * s.N * 4)};
            cuuint32_t yb[3] = {32, 32, 1};
            cuuint32_t ye[3] = {1, 1, 1};
            ok = encode_f32(&ty, c.y, 3, yd, ys, yb, ye);
        }
        if (!ok) return cudaErrorInvalidValue;
    }
    p.mp_tiles = (p.m_tiles + CG - 1) / CG;
    if constexpr (TQ == 128) p.mp_tiles = (int)s.n * p.tiles_q * ((p.P + CG - 1) / CG);  // pairs split the rows
    const long long tiles = (long long)p.batch * p.mp_tiles * p.n_tiles;
    const long long units = tiles * c.split;
    if (units >= (1ll << 31)) return cudaErrorInvalidValue;
    p.units = (int)units;
    p.sched = c.sched;
    p.raster = c.raster;
    p.epi = c.epi == 2 ? 2 : 1;
    p.total_iters = tiles * p.kblocks;
    if (c.split > 1) {
        cudaError_t e = zero_for_splitk((float*)c.y, s.y_elems, c.stream);
        if (e != cudaSuccess) return e;
    }
    // persistent grid: as many CTA groups as can be co-resident (the stream-K flag protocol
    // spins heads on their tails, so every group MUST be resident at once): the occupancy
    // calculator's active clusters (registers, shared memory, cluster shape) capped by TMEM
    const int stages = c.stages;
    const int b_res = TQ == 128 ? p.CB * p.R * p.S * Cfg::B_BYTES : 0;
    const size_t smem = tc_smem_bytes<BN, BK, TQ, CG, EW>(stages, p.a_stage_bytes, b_res);
    if (stages < 2 || stages > Cfg::MAX_STAGES || smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    p.stages = stages;
    const long long groups_max = tc_resident_groups<BN, BK, TQ, CG, EW>(c.num_sms, stages, p.a_stage_bytes, b_res);
    if (groups_max < 1) return cudaErrorInvalidConfiguration;
    long long groups = groups_max;
    if (c.sched >= 1) {
        if (!c.sk || !c.sk->flags || !c.sk->ws) return cudaErrorInvalidValue;  // the handle owns the workspace
        p.flags = c.sk->flags;
        p.ws = c.sk->ws;
        if (groups > p.total_iters) groups = p.total_iters;
        if (groups * CG > c.sk->slots) groups = c.sk->slots / CG;
        if (c.sched == 2) {  // whole waves tile by tile; the remainder tiles cut into equal k-chunks,
                             // one chunk per group (groups without one stop after their waves)
            p.dp_tiles = (int)((tiles / groups) * groups);
            p.rem_tiles = (int)(tiles - p.dp_tiles);
            long long S = p.rem_tiles ? groups / p.rem_tiles : 1;
            if (S < 1) S = 1;
            if (S > p.kblocks) S = p.kblocks;
            p.rem_chunks = (int)S;
            p.total_iters = (long long)p.rem_tiles * p.kblocks;
        }
    } else if (groups > units) {
        groups = units;
    }
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)(groups * CG));
    cfg.blockDim = dim3(Cfg::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    pdl_attr(attr[1]);  // launch early: the prologue overlaps the preceding kernel's tail
    cfg.numAttrs = 2;
    static const bool tracing = std::getenv("DB200_TC_TRACE") != nullptr;
    static unsigned long long* trace_buf = nullptr;
    if (tracing && !trace_buf && cudaMalloc(&trace_buf, 4096 * 16 * sizeof(unsigned long long)) != cudaSuccess)
        trace_buf = nullptr;
    p.trace = tracing ? trace_buf : nullptr;
    if (p.trace) cudaMemsetAsync(p.trace, 0, (size_t)cfg.gridDim.x * 16 * sizeof(unsigned long long), c.stream);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, ty, p);
    count_launches(1);
    if (p.trace && e == cudaSuccess) {  // debug: per-CTA timeline in microseconds from the earliest start
        std::vector<unsigned long long> h((size_t)cfg.gridDim.x * 16);
        cudaStreamSynchronize(c.stream);
        cudaMemcpy(h.data(), p.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (unsigned i = 0; i < cfg.gridDim.x; ++i) t0 = std::min(t0, h[i * 16]);
        std::fprintf(stderr, "TC_TRACE sched %d groups %lld tiles %lld dp %d rem %d chunks %d\n", p.sched, groups,
                     tiles, p.dp_tiles, p.rem_tiles, p.rem_chunks);
        for (unsigned i = 0; i < cfg.gridDim.x; i += CG) {
            std::fprintf(stderr, "cta %3u:", i);
            for (int k = 0; k < 16; ++k)
                std::fprintf(stderr, " %7.2f", h[i * 16 + k] ? (h[i * 16 + k] - t0) * 1e-3 : -1.0);
            std::fprintf(stderr, "\n");
        }
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

constexpr bool tc_static_ok(int BN, int BK, int CG) {  // at least a 2-stage ring fits
    return 1024 + (size_t)2 * (128 + BN / CG) * BK * 2 + 256 + kTcEpiBytes <= 227 * 1024;
}

template <int BN, int BK, int TQ, int CG>
void tc_register() {  // key: (sketch, BM, BN, BK, EW, TILE_Q); STAGES is a runtime knob
    if constexpr (tc_static_ok(BN, BK, CG)) {
        registry_add(kernel_key(TQ ? SK_TC_IGEMM_CONV_BF16 : SK_TC_GEMM_BF16, 128 * CG, BN, BK, 4, TQ),
                     &tc_launch<BN, BK, TQ, CG, 4>);
        registry_add(kernel_key(TQ ? SK_TC_IGEMM_CONV_BF16 : SK_TC_GEMM_BF16, 128 * CG, BN, BK, 8, TQ),
                     &tc_launch<BN, BK, TQ, CG, 8>);
    }
}

#define TC_SHAPES(TQ, CG)                                                                                        \
    tc_register<64, 64, TQ, CG>(); tc_register<128, 64, TQ, CG>(); tc_register<192, 64, TQ, CG>();             \
    tc_register<256, 64, TQ, CG>(); tc_register<64, 128, TQ, CG>(); tc_register<128, 128, TQ, CG>();           \
    tc_register<192, 128, TQ, CG>(); tc_register<256, 128, TQ, CG>();

void register_tc_gemm() {
    TC_SHAPES(0, 1) TC_SHAPES(0, 2)     // dense / bmm
    TC_SHAPES(8, 1) TC_SHAPES(8, 2)     // conv, 16 x 8 pixel sub-tiles
    TC_SHAPES(16, 1) TC_SHAPES(16, 2)   // conv, 8 x 16
    TC_SHAPES(32, 1) TC_SHAPES(32, 2)   // conv, 4 x 32
    // conv, halo row tiles of 128 pixels (BK = 64: one channel block of the R input-row windows)
    tc_register<64, 64, 128, 1>(); tc_register<128, 64, 128, 1>(); tc_register<192, 64, 128, 1>();
    tc_register<256, 64, 128, 1>(); tc_register<64, 64, 128, 2>(); tc_register<128, 64, 128, 2>();
    tc_register<192, 64, 128, 2>(); tc_register<256, 64, 128, 2>();
}

}  // namespace db200
