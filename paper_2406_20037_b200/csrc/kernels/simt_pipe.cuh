// simt_pipe.cuh — sketches SIMT_PIPE_GEMM_F32 and SIMT_PIPE_CONV_F32.
//
// The same loop nest as simt_gemm.cuh (Def. 2.1: Y[m,n] = sum_k A[m,k] B[n,k],
// m/n split into BM x BN block tiles, TT x TT register tiles, k split into BK steps), with
// a different staging and reduction structure, aimed at the small batch-1 layers whose
// CTAs own only a few k-tiles and so never amortise one global-load latency per tile:
//
//   * cp.async multistage staging: a STAGES-deep ring of [BM][BK] / [BN][BK] shared-memory
//     tiles filled by cp.async (16-byte copies for VEC = 4, 4-byte for VEC = 1) with
//     zero-fill for padding taps and ragged edges, so STAGES-1 tiles are in flight while
//     one is consumed (north_star: "TMA or cp.async shared-memory staging");
//   * sliced K inside the CTA: KW warp groups own disjoint k sub-ranges of every staged tile
//     (BK/KW each) and are summed through shared memory at the end -- more warps per output
//     tile without split-K's global atomics and zeroing launch;
//   * k-parity FFMA2: each accumulator is a float2 of (even-k, odd-k) partial sums, so
//     fma.rn.f32x2 takes both operands straight from the float4 shared-memory loads
//     (no broadcast repacking); the two halves are added in the epilogue.
//
// Annotations: BM, BN, BK, TT, KW (compile-time); VEC, STAGES, SPLIT_K (runtime).
// CONV = true is the implicit-GEMM view of conv2d (NHWC x KRSC -> NPQK, R-C2); the
// (r, s, c) decomposition of every reduction index of the CTA's k range is tabulated once
// in shared memory, a gathered element is X[row base + koff(kk)] when its tap is inside the
// image, else zero (cp.async src-size 0).
#pragma once
#include "common.cuh"

namespace db200 {

struct PipeParams {
    const float* __restrict__ A;
    const float* __restrict__ B;
    float* __restrict__ C;
    int M, N, K;
    long long sA, sB, sC;  // batch strides
    int ktiles, kt_per_split, split;
    int H, W, Cin, P, Q, S, sh, sw, ph, pw, dh, dw;
    int vw;      // VEC knob: elements per cp.async (4 or 1)
    int stages;  // STAGES knob
    // work units: (k slice, m tile, n tile, batch), k slice fastest; a CTA takes units
    // blockIdx.x, + gridDim.x, ... (one unit per CTA when OCC = 0, persistent otherwise)
    int units, m_tiles, n_tiles;
    int persist;  // 1: the k table covers all of K and the epilogue tile has its own smem
    int cred;     // 1: the SPLIT_K CTAs of a tile form a cluster and reduce their partial tiles
                  //    through distributed shared memory (no zeroing kernel, no atomics)
};

constexpr bool pipe_static_ok(int BM, int BN, int BK, int TT, int KW) {
    return TT <= BM && TT <= BN && (BM / TT) * (BN / TT) >= 32 && (BM / TT) * (BN / TT) * KW <= 1024 &&
           BK % (4 * KW) == 0;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_wait_stages(int stages) {  // wait until <= STAGES-2 groups pending
    switch (stages) {
        case 2: cp_wait<0>(); break;
        case 3: cp_wait<1>(); break;
        case 4: cp_wait<2>(); break;
        default: cp_wait<4>(); break;  // 6
    }
}

__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// (a.x*b.x + c.x, a.y*b.y + c.y): two RN fused multiply-adds in one FFMA2
__device__ __forceinline__ float2 ffma2_ew(float2 a, float2 b, float2 c) {
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return r;
}

template <int BM, int BN, int BK, int TT, int KW, int VW, bool CONV>
__global__ void __launch_bounds__((BM / TT) * (BN / TT) * KW) simt_pipe_kernel(const PipeParams p) {
    constexpr int TX = BN / TT, TY = BM / TT, GT = TX * TY, NT = GT * KW, LDK = BK + 4, BKG = BK / KW;
    extern __shared__ __align__(16) float smem[];
    const int stages = p.stages;
    float* ring = smem;  // [stages][(BM + BN) * LDK]
    constexpr int STAGE_FLOATS = (BM + BN) * LDK;
    const size_t pipe_floats = (size_t)stages * STAGE_FLOATS;
    const bool staged_epi = KW > 1 || p.split > 1;  // epilogue through shared memory
    const size_t red_floats = staged_epi ? (size_t)KW * BM * pipe_red_ld(BN) : 0;
    // one-unit CTAs stage the epilogue tile over the drained ring; persistent CTAs keep the
    // next unit's tiles in flight during an epilogue, so their tile has its own region
    float* red = p.persist ? smem + pipe_floats : smem;
    const size_t head = p.persist ? pipe_floats + red_floats : (pipe_floats > red_floats ? pipe_floats : red_floats);
    int2* ktab = reinterpret_cast<int2*>(smem + head);

    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid % GT;
    // a warp covers an 8 x 4 (or 4 x 8) patch of the thread grid: its fragment loads touch 8
    // B rows and 4 A rows (4 and 8), one 128-byte shared-memory wavefront each, where a
    // 16 x 2 or 32 x 1 patch needs 2-4 wavefronts per B load
    int tx, ty;
    if constexpr (TX % 8 == 0 && TY % 4 == 0) {
        const int lane = gt & 31, wi = gt >> 5;
        tx = (wi % (TX / 8)) * 8 + (lane & 7);
        ty = (wi / (TX / 8)) * 4 + (lane >> 3);
    } else if constexpr (TX % 4 == 0 && TY % 8 == 0) {
        const int lane = gt & 31, wi = gt >> 5;
        tx = (wi % (TX / 4)) * 4 + (lane & 3);
        ty = (wi / (TX / 4)) * 8 + (lane >> 2);
    } else {
        tx = gt % TX;
        ty = gt / TX;
    }
    constexpr int RLD = pipe_red_ld(BN);  // staged epilogue tile row stride (floats)
    constexpr int CPR = BK / VW;  // cp.async chunks per tile row
    const int u0 = blockIdx.x, ustep = gridDim.x;
    // programmatic dependent launch: the next kernel in the stream may start its own prologue now
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (u0 >= p.units) return;

    // unit -> (k slice, m tile, n tile, batch), k slice fastest
    struct Unit {
        int m0, n0, bz, kt_begin, nk;
    };
    auto unit_of = [&](int u) {
        Unit w;
        const int kz = u % p.split;
        int t = u / p.split;
        w.m0 = (t % p.m_tiles) * BM;
        t /= p.m_tiles;
        w.n0 = (t % p.n_tiles) * BN;
        w.bz = t / p.n_tiles;
        w.kt_begin = kz * p.kt_per_split;
        w.nk = min(p.ktiles, w.kt_begin + p.kt_per_split) - w.kt_begin;  // >= 1 (static validity)
        return w;
    };

    // the conv k table: koff / tap offsets of every reduction chunk, for the CTA's k range
    // (one unit) or for all of K (persistent: units of every k slice)
    const Unit first = unit_of(u0);
    const int ktab_k0 = p.persist ? 0 : first.kt_begin * BK;
    if constexpr (CONV) {
        const int nent = p.persist ? (p.ktiles * BK) / VW : (first.nk * BK) / VW;
        for (int j = tid; j < nent; j += NT) {
            const int kk = ktab_k0 + j * VW;
            int2 t = make_int2(0, 0x7FFF7FFF);  // out of range: fails the image bounds check
            if (kk < p.K) {
                const int rs = kk / p.Cin, c = kk - rs * p.Cin, r = rs / p.S, s = rs - r * p.S;
                const int dr = r * p.dh, ds = s * p.dw;
                t = make_int2((dr * p.W + ds) * p.Cin + c, (dr << 16) | ds);
            }
            ktab[j] = t;
        }
        __syncthreads();
    }

    // per-slot producer state of the unit being loaded: a slot is (row, k chunk) of the tile,
    // the same for every k-tile of a unit
    constexpr int chunksA = BM * CPR, chunksB = BN * CPR;
    constexpr int SA = (chunksA + NT - 1) / NT, SB = (chunksB + NT - 1) / NT;  // slots per thread
    static_assert(SA <= kPipeMaxSlots && SB <= kPipeMaxSlots, "slot budget (static validity rule)");
    int abase[SA], ah0[SA], aw0[SA];  // A: image / row base, h0, w0 (conv) or row offset (dense; h0 = 0 = valid)
    int boff[SB];                     // B: element offset of the row (-1: row outside N)
    const float* Ab = p.A;
    const float* Bb = p.B;
    Unit lw = first;  // the unit the producer is loading
    auto set_unit = [&](const Unit& w) {
        Ab = p.A + (CONV ? 0 : w.bz * p.sA);
        Bb = p.B + w.bz * p.sB;
#pragma unroll
        for (int i = 0; i < SA; ++i) {
            const int e = tid + i * NT;
            const int row = e / CPR;
            int base = 0, h0 = -(1 << 29), w0 = 0;
            if (e < chunksA && w.m0 + row < p.M) {
                const int m = w.m0 + row;
                if constexpr (CONV) {
                    const int q = m % p.Q, t = m / p.Q, pp = t % p.P, n = t / p.P;
                    h0 = pp * p.sh - p.ph;
                    w0 = q * p.sw - p.pw;
                    base = n * p.H * p.W * p.Cin + (h0 * p.W + w0) * p.Cin;
                } else {
                    base = m * p.K;
                    h0 = 0;
                }
            }
            abase[i] = base; ah0[i] = h0; aw0[i] = w0;
        }
#pragma unroll
        for (int i = 0; i < SB; ++i) {
            const int e = tid + i * NT, row = e / CPR;
            boff[i] = (e < chunksB && w.n0 + row < p.N) ? (w.n0 + row) * p.K : -1;
        }
    };
    set_unit(lw);

    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    auto load_tile = [&](int stage, int kt) {  // kt relative to the loaded unit's first k-tile
        const uint32_t as = ring_s + (uint32_t)(stage * STAGE_FLOATS) * 4u;
        const uint32_t bs = as + (uint32_t)(BM * LDK) * 4u;
        const int kb = (lw.kt_begin + kt) * BK;  // absolute k of the tile
#pragma unroll
        for (int i = 0; i < SA; ++i) {
            const int e = tid + i * NT;
            if (chunksA % NT == 0 || e < chunksA) {
                const int row = e / CPR, kl = (e % CPR) * VW;
                const uint32_t dst = as + (uint32_t)(row * LDK + kl) * 4u;
                // branch-free: an out-of-image tap copies 0 bytes from the tensor base
                int ok, off;
                if constexpr (CONV) {
                    const int2 t = ktab[(kb - ktab_k0 + kl) / VW];
                    const int h = ah0[i] + (t.y >> 16), w = aw0[i] + (t.y & 0xFFFF);
                    ok = (unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W;
                    off = ok ? abase[i] + t.x : 0;
                } else {
                    const int kk = kb + kl;
                    ok = ah0[i] == 0 && kk < p.K;
                    off = ok ? abase[i] + kk : 0;
                }
                const float* src = Ab + off;
                if constexpr (VW == 4) cp_async16(dst, src, ok ? 16 : 0);
                else cp_async4(dst, src, ok ? 4 : 0);
            }
        }
#pragma unroll
        for (int i = 0; i < SB; ++i) {
            const int e = tid + i * NT;
            if (chunksB % NT == 0 || e < chunksB) {
                const int row = e / CPR, kl = (e % CPR) * VW;
                const uint32_t dst = bs + (uint32_t)(row * LDK + kl) * 4u;
                const bool ok = boff[i] >= 0 && kb + kl < p.K;
                const float* src = Bb + (ok ? boff[i] + kb + kl : 0);
                if constexpr (VW == 4) cp_async16(dst, src, ok ? 16 : 0);
                else cp_async4(dst, src, ok ? 4 : 0);
            }
        }
    };

    float2 acc[TT][TT];
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TT; ++j) acc[i][j] = make_float2(0.f, 0.f);

    auto compute = [&](int stage) {
        const float* as = ring + stage * STAGE_FLOATS + ty * LDK + g * BKG;
        const float* bs = ring + stage * STAGE_FLOATS + BM * LDK + tx * LDK + g * BKG;
        constexpr int NKQ = BKG / 4;
        // register double buffer: the fragments of step kq+1 are loaded before the FFMA2s of
        // step kq, so shared-memory latency overlaps the math within one warp
        float4 a4[2][TT], b4[2][TT];
#pragma unroll
        for (int i = 0; i < TT; ++i) a4[0][i] = *reinterpret_cast<const float4*>(as + i * TY * LDK);
#pragma unroll
        for (int j = 0; j < TT; ++j) b4[0][j] = *reinterpret_cast<const float4*>(bs + j * TX * LDK);
#pragma unroll
        for (int kq = 0; kq < NKQ; ++kq) {
            const int cur = kq & 1;
            if (kq + 1 < NKQ) {
#pragma unroll
                for (int i = 0; i < TT; ++i)
                    a4[cur ^ 1][i] = *reinterpret_cast<const float4*>(as + i * TY * LDK + (kq + 1) * 4);
#pragma unroll
                for (int j = 0; j < TT; ++j)
                    b4[cur ^ 1][j] = *reinterpret_cast<const float4*>(bs + j * TX * LDK + (kq + 1) * 4);
            }
            // two passes (k, k+1) then (k+2, k+3): TT*TT independent FFMA2 between the two
            // updates of one accumulator
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
                for (int j = 0; j < TT; ++j)
                    acc[i][j] = ffma2_ew(make_float2(a4[cur][i].x, a4[cur][i].y),
                                         make_float2(b4[cur][j].x, b4[cur][j].y), acc[i][j]);
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
                for (int j = 0; j < TT; ++j)
                    acc[i][j] = ffma2_ew(make_float2(a4[cur][i].z, a4[cur][i].w),
                                         make_float2(b4[cur][j].z, b4[cur][j].w), acc[i][j]);
        }
    };

    const bool atomic = p.split > 1 && !p.cred;
    // split-K inside a cluster (RED = 1): the split CTAs of a tile are one cluster; each stages
    // its partial tile (KW groups summed) in shared memory, and after a cluster barrier CTA r
    // sums rows [r*BM/S, (r+1)*BM/S) of all S partial tiles over distributed shared memory
    // (ld.shared::cluster) and stores them -- Y written once, in order-independent of timing
    auto epilogue_cluster = [&](const Unit& w) {
        float* __restrict__ C = p.C + w.bz * p.sC;
        cp_wait<0>();
        __syncthreads();  // the ring is drained; the tile overlaps it
#pragma unroll
        for (int i = 0; i < TT; ++i)
#pragma unroll
            for (int j = 0; j < TT; ++j)
                red[(g * BM + ty + i * TY) * RLD + tx + j * TX] = acc[i][j].x + acc[i][j].y;
        if constexpr (KW > 1) {
            __syncthreads();
            for (int e = tid; e < BM * BN / 4; e += NT) {
                const int o = (e / (BN / 4)) * RLD + (e % (BN / 4)) * 4;
                float4 v = *reinterpret_cast<const float4*>(red + o);
#pragma unroll
                for (int q = 1; q < KW; ++q) {
                    const float4 u = *reinterpret_cast<const float4*>(red + q * BM * RLD + o);
                    v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
                }
                *reinterpret_cast<float4*>(red + o) = v;
            }
        }
        cluster_barrier();  // every CTA's partial tile is in its shared memory
        const int S = p.split;
        uint32_t rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        const int rp = (BM + S - 1) / S, r0 = (int)rank * rp, r1 = min(BM, r0 + rp);
        const uint32_t red_s = (uint32_t)__cvta_generic_to_shared(red);
        const bool vec_ok = (p.N % 4) == 0;
        for (int e = r0 * (BN / 4) + tid; e < r1 * (BN / 4); e += NT) {
            const int row = e / (BN / 4), col = (e % (BN / 4)) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < S; ++q) {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(red_s + (uint32_t)(row * RLD + col) * 4u), "r"(q));
                float4 u;
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(u.x), "=f"(u.y), "=f"(u.z), "=f"(u.w) : "r"(ra) : "memory");
                v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
            }
            const int m = w.m0 + row, n = w.n0 + col;
            if (m >= p.M) continue;
            float* cp = C + (long long)m * p.N + n;
            if (vec_ok && n + 3 < p.N) {
                *reinterpret_cast<float4*>(cp) = v;
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (n + q < p.N) cp[q] = vv[q];
            }
        }
        cluster_barrier();  // no CTA leaves while its peers still read its shared memory
    };

    // epilogue of the unit `w` the consumer just finished: its accumulators -> Y
    auto epilogue = [&](const Unit& w) {
        if (p.cred) return epilogue_cluster(w);
        float* __restrict__ C = p.C + w.bz * p.sC;
        if (atomic) griddep_wait();  // Y zeroed by the prerequisite grid (PDL); returns at once later
        if (!staged_epi) {  // KW = 1, no split-K: direct stores from the accumulators
#pragma unroll
            for (int i = 0; i < TT; ++i) {
                const int m = w.m0 + ty + i * TY;
                if (m >= p.M) continue;
                float* crow = C + (long long)m * p.N;
#pragma unroll
                for (int j = 0; j < TT; ++j) {
                    const int n = w.n0 + tx + j * TX;
                    if (n < p.N) crow[n] = acc[i][j].x + acc[i][j].y;
                }
            }
            return;
        }
        // the KW groups' partial tiles summed through shared memory; 128-bit stores or
        // (split-K) 128-bit atomics from the staged tile
        if (!p.persist) cp_wait<0>();  // the tile overlaps the (drained) ring
        __syncthreads();               // every thread is done reading the previous staged tile
#pragma unroll
        for (int i = 0; i < TT; ++i)
#pragma unroll
            for (int j = 0; j < TT; ++j)
                red[(g * BM + ty + i * TY) * RLD + tx + j * TX] = acc[i][j].x + acc[i][j].y;
        __syncthreads();
        const bool vec_ok = (p.N % 4) == 0;
        for (int e = tid; e < BM * BN / 4; e += NT) {
            const int row = e / (BN / 4), col = (e % (BN / 4)) * 4;
            const int m = w.m0 + row, n = w.n0 + col;
            if (m >= p.M) continue;
            float4 v = *reinterpret_cast<const float4*>(red + row * RLD + col);
#pragma unroll
            for (int q = 1; q < KW; ++q) {
                const float4 u = *reinterpret_cast<const float4*>(red + (q * BM + row) * RLD + col);
                v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
            }
            float* cp = C + (long long)m * p.N + n;
            if (vec_ok && n + 3 < p.N) {
                if (atomic) atomicAdd(reinterpret_cast<float4*>(cp), v);
                else *reinterpret_cast<float4*>(cp) = v;
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (n + q < p.N) {
                        if (atomic) atomicAdd(cp + q, vv[q]);
                        else cp[q] = vv[q];
                    }
            }
        }
    };

    // multistage ring over the concatenated k-tiles of this CTA's units: STAGES-1 tiles in
    // flight while one is consumed; a persistent CTA's producer runs into the next unit's
    // tiles while the consumer finishes the current one (no pipeline drain between units)
    int lu = u0, lkt = 0;  // producer cursor: unit, k-tile within it
    auto produce = [&](int stage) {
        if (lu >= p.units) return;
        load_tile(stage, lkt);
        if (++lkt == lw.nk) {
            lkt = 0;
            lu += ustep;
            if (lu < p.units) {
                lw = unit_of(lu);
                set_unit(lw);
            }
        }
    };
    // Launched with programmatic stream serialization: the prologue above (k table, slot setup)
    // overlaps the preceding kernel's tail.  X and W are read only after that kernel completed --
    // except behind this schedule's own split-K zeroing kernel (plainly serialised, so every
    // earlier kernel is complete when it starts), where the wait is deferred to the first atomic.
    if (!atomic) griddep_wait();
    for (int s = 0; s < stages - 1; ++s) {
        produce(s);
        cp_commit();
    }
    Unit cw = first;  // the unit the consumer is computing
    int ckt = 0;
    int cs = 0, ls = stages - 1;  // stage consumed / stage refilled this iteration (no modulo)
    for (int cu = u0; cu < p.units;) {
        cp_wait_stages(stages);
        __syncthreads();  // tile visible to all; every thread is done with the previous tile's stage
        produce(ls);
        cp_commit();
        compute(cs);
        cs = cs + 1 == stages ? 0 : cs + 1;
        ls = ls + 1 == stages ? 0 : ls + 1;
        if (++ckt == cw.nk) {
            epilogue(cw);
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
                for (int j = 0; j < TT; ++j) acc[i][j] = make_float2(0.f, 0.f);
            ckt = 0;
            cu += ustep;
            if (cu < p.units) cw = unit_of(cu);
        }
    }
}

template <int BM, int BN, int BK, int TT, int KW, int VW, bool CONV>
cudaError_t pipe_launch(const LaunchCtx& c) {
    constexpr int NT = (BM / TT) * (BN / TT) * KW;
    auto kern = simt_pipe_kernel<BM, BN, BK, TT, KW, VW, CONV>;
    static std::atomic<unsigned long long> optin{0};
    {
        cudaError_t e = smem_optin(optin, kern, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const ShapeInfo& s = *c.sh;
    PipeParams p;
    p.A = (const float*)c.x;
    p.B = (const float*)c.w;
    p.C = (float*)c.y;
    p.M = (int)s.M; p.N = (int)s.N; p.K = (int)s.K;
    p.sA = s.M * s.K; p.sB = s.N * s.K; p.sC = s.M * s.N;
    p.ktiles = (int)((s.K + BK - 1) / BK);
    p.split = c.split;
    p.kt_per_split = (p.ktiles + c.split - 1) / c.split;
    p.H = (int)s.h; p.W = (int)s.w; p.Cin = (int)s.c; p.P = (int)s.p; p.Q = (int)s.q; p.S = (int)s.s;
    p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
    p.vw = VW;
    p.stages = c.stages;
    p.m_tiles = (int)((s.M + BM - 1) / BM);
    p.n_tiles = (int)((s.N + BN - 1) / BN);
    const long long units = (long long)p.m_tiles * p.n_tiles * s.batch * c.split;
    if (units >= (1ll << 31)) return cudaErrorInvalidValue;
    p.units = (int)units;
    // OCC knob: 0 = one CTA per unit; k > 0 = persistent, k CTAs per SM walking the units
    long long grid = units;
    p.persist = 0;
    if (c.occ > 0 && units > (long long)c.occ * c.num_sms) {
        grid = (long long)c.occ * c.num_sms;
        p.persist = 1;
    }
    // RED knob: 1 = split-K reduced inside a cluster of the tile's SPLIT_K CTAs (k slice
    // fastest, so consecutive CTAs = one tile's slices = one cluster)
    p.cred = (c.red == 1 && c.split > 1 && !p.persist) ? 1 : 0;
    if (c.red == 1 && !p.cred) return cudaErrorInvalidConfiguration;
    if (c.split > 1 && !p.cred) {
        cudaError_t e = zero_for_splitk((float*)c.y, s.y_elems, c.stream);
        if (e != cudaSuccess) return e;
    }
    const size_t smem = pipe_smem_bytes(BM, BN, BK, KW, p.stages, CONV, p.persist ? p.ktiles * BK : p.kt_per_split * BK,
                                        p.vw, p.split, p.persist);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    // always a programmatic dependent launch (after the zeroing kernel, the kernel waits before
    // its first atomic; otherwise before its first load)
    cudaLaunchAttribute attr[2];
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p.cred) {
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = (unsigned)c.split;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.numAttrs = 2;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    count_launches(1);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int BM, int BN, int BK, int TT, int KW, bool CONV>
void pipe_register() {
    if constexpr (pipe_static_ok(BM, BN, BK, TT, KW)) {  // VEC is compiled too: key field = KW | VEC << 4
        constexpr int32_t sk = CONV ? SK_SIMT_PIPE_CONV_F32 : SK_SIMT_PIPE_GEMM_F32;
        constexpr int NT = (BM / TT) * (BN / TT) * KW;
        registry_add(kernel_key(sk, BM, BN, BK, TT, KW | (4 << 4)), &pipe_launch<BM, BN, BK, TT, KW, 4, CONV>);
        if constexpr ((BM * BK + NT - 1) / NT <= kPipeMaxSlots && (BN * BK + NT - 1) / NT <= kPipeMaxSlots)
            registry_add(kernel_key(sk, BM, BN, BK, TT, KW | (1 << 4)), &pipe_launch<BM, BN, BK, TT, KW, 1, CONV>);
    }
}

}  // namespace db200
