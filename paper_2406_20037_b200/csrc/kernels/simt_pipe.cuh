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
    const size_t red_floats = staged_epi ? (size_t)KW * BM * BN : 0;
    int2* ktab = reinterpret_cast<int2*>(smem + (pipe_floats > red_floats ? pipe_floats : red_floats));

    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid % GT;
    const int tx = gt % TX, ty = gt / TX;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int bz = blockIdx.z / p.split, kz = blockIdx.z % p.split;
    const int kt_begin = kz * p.kt_per_split;
    const int kt_end = min(p.ktiles, kt_begin + p.kt_per_split);
    if (kt_begin >= kt_end) return;
    const int nk = kt_end - kt_begin;
    constexpr int CPR = BK / VW;  // cp.async chunks per tile row
    const int kbeg = kt_begin * BK;

    const float* __restrict__ A = p.A + (CONV ? 0 : bz * p.sA);
    const float* __restrict__ B = p.B + bz * p.sB;
    float* __restrict__ C = p.C + bz * p.sC;

    // per-slot fixed state: a slot is (row, k chunk) of the tile, the same for every k-tile
    constexpr int chunksA = BM * CPR, chunksB = BN * CPR;
    constexpr int SA = (chunksA + NT - 1) / NT, SB = (chunksB + NT - 1) / NT;  // slots per thread
    static_assert(SA <= kPipeMaxSlots && SB <= kPipeMaxSlots, "slot budget (static validity rule)");
    // A slots: image / row base, h0, w0 (conv) or row offset (dense; h0 = 0 marks a valid row)
    int abase[SA], ah0[SA], aw0[SA];
#pragma unroll
    for (int i = 0; i < SA; ++i) {
        const int e = tid + i * NT;
        const int row = e / CPR;
        int base = 0, h0 = -(1 << 29), w0 = 0;
        if (e < chunksA && m0 + row < p.M) {
            const int m = m0 + row;
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
    if constexpr (CONV) {  // koff / tap offsets of every reduction chunk in this CTA's k range
        const int nent = (nk * BK) / VW;
        for (int j = tid; j < nent; j += NT) {
            const int kk = kbeg + j * VW;
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

    // B slots: element offset of the slot's first k in this CTA's range (-1: row outside N)
    int boff[SB];
#pragma unroll
    for (int i = 0; i < SB; ++i) {
        const int e = tid + i * NT, row = e / CPR, kl = (e % CPR) * VW;
        boff[i] = (e < chunksB && n0 + row < p.N) ? (n0 + row) * p.K + kbeg + kl : -1;
    }

    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    auto load_tile = [&](int stage, int kt) {  // kt relative to kt_begin
        const uint32_t as = ring_s + (uint32_t)(stage * STAGE_FLOATS) * 4u;
        const uint32_t bs = as + (uint32_t)(BM * LDK) * 4u;
        const int k0 = kt * BK;  // local k offset
#pragma unroll
        for (int i = 0; i < SA; ++i) {
            const int e = tid + i * NT;
            if (chunksA % NT == 0 || e < chunksA) {
                const int row = e / CPR, kl = (e % CPR) * VW;
                const uint32_t dst = as + (uint32_t)(row * LDK + kl) * 4u;
                // branch-free: an out-of-image tap copies 0 bytes from the tensor base
                int ok, off;
                if constexpr (CONV) {
                    const int2 t = ktab[(k0 + kl) / VW];
                    const int h = ah0[i] + (t.y >> 16), w = aw0[i] + (t.y & 0xFFFF);
                    ok = (unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W;
                    off = ok ? abase[i] + t.x : 0;
                } else {
                    const int kk = kbeg + k0 + kl;
                    ok = ah0[i] == 0 && kk < p.K;
                    off = ok ? abase[i] + kk : 0;
                }
                const float* src = A + off;
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
                const bool ok = boff[i] >= 0 && kbeg + k0 + kl < p.K;
                const float* src = B + (ok ? boff[i] + k0 : 0);
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

    // multistage ring: STAGES-1 tiles in flight while one is consumed
    for (int s = 0; s < stages - 1; ++s) {
        if (s < nk) load_tile(s, s);
        cp_commit();
    }
    int cs = 0, ls = stages - 1;  // stage consumed / stage refilled this iteration (no modulo)
    for (int it = 0; it < nk; ++it) {
        cp_wait_stages(stages);
        __syncthreads();  // tile `it` visible to all; every thread is done with tile it-1's stage
        const int nxt = it + stages - 1;
        if (nxt < nk) load_tile(ls, nxt);
        cp_commit();
        compute(cs);
        cs = cs + 1 == stages ? 0 : cs + 1;
        ls = ls + 1 == stages ? 0 : ls + 1;
    }

    const bool atomic = p.split > 1;
    if (atomic) griddep_wait();  // Y zeroed by the prerequisite grid (PDL)
    if (!staged_epi) {  // KW = 1, no split-K: direct stores from the accumulators
#pragma unroll
        for (int i = 0; i < TT; ++i) {
            const int m = m0 + ty + i * TY;
            if (m >= p.M) continue;
            float* crow = C + (long long)m * p.N;
#pragma unroll
            for (int j = 0; j < TT; ++j) {
                const int n = n0 + tx + j * TX;
                if (n < p.N) {
                    const float v = acc[i][j].x + acc[i][j].y;
                    if (atomic) atomicAdd(crow + n, v);
                    else crow[n] = v;
                }
            }
        }
    } else {  // the KW groups' partial tiles summed through shared memory; 128-bit stores or
              // (split-K) 128-bit atomics from the staged tile
        cp_wait<0>();
        __syncthreads();
        float* red = smem;  // [KW][BM][BN]
#pragma unroll
        for (int i = 0; i < TT; ++i)
#pragma unroll
            for (int j = 0; j < TT; ++j)
                red[(g * BM + ty + i * TY) * BN + tx + j * TX] = acc[i][j].x + acc[i][j].y;
        __syncthreads();
        const bool vec_ok = (p.N % 4) == 0;
        for (int e = tid; e < BM * BN / 4; e += NT) {
            const int row = e / (BN / 4), col = (e % (BN / 4)) * 4;
            const int m = m0 + row, n = n0 + col;
            if (m >= p.M) continue;
            float4 v = *reinterpret_cast<const float4*>(red + row * BN + col);
#pragma unroll
            for (int q = 1; q < KW; ++q) {
                const float4 u = *reinterpret_cast<const float4*>(red + (q * BM + row) * BN + col);
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
    if (c.split > 1) {
        cudaError_t e = zero_for_splitk((float*)c.y, s.y_elems, c.stream);
        if (e != cudaSuccess) return e;
    }
    const size_t smem = pipe_smem_bytes(BM, BN, BK, KW, p.stages, CONV, p.kt_per_split * BK, p.vw, p.split);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((s.M + BM - 1) / BM), (unsigned)((s.N + BN - 1) / BN), (unsigned)(s.batch * c.split));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    if (c.split > 1) {  // launch early; the kernel waits for the zeroing before its atomics
        pdl_attr(attr[0]);
        cfg.attrs = attr;
        cfg.numAttrs = 1;
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
