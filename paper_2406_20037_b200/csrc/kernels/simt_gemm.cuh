// simt_gemm.cuh — sketches SIMT_GEMM_F32 and SIMT_IGEMM_CONV_F32.
//
// One fixed sequence of transformations (a "sketch", Def. 2.1) of
// the naive loop nest Y[m,n] = sum_k A[m,k] B[n,k]: split m and n into BM x BN
// block tiles bound to CTAs, split each block tile into TT x TT register tiles
// bound to threads, split k into BK-wide steps staged through shared memory,
// unroll the inner k loop by UNROLL, and optionally split the k range across
// SPLIT_K CTAs whose partial sums are reduced with vector atomics.
// Annotations (the knobs): BM, BN, BK, TT, UNROLL (compile-time), VEC (global
// load width: 1 = scalar, 4 = 128-bit), STAGES (shared-memory staging depth:
// 1 = load/sync/compute, 2 = the next tile's global loads are issued into
// registers before this tile's FMAs), SPLIT_K (runtime).
//
// CONV = true is the implicit-GEMM view of conv2d (NHWC x KRSC -> NPQK):
// A[m, kk] = X[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c] with m = (n,p,q), kk = (r,s,c),
// gathered on the fly (zero outside the image); B = W viewed as [K][R*S*C].
//
// FP32 on the CUDA cores (north_star: "The fp32 SIMT variants stay on CUDA cores").
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"

namespace db200 {

struct SimtParams {
    const void* __restrict__ A;  // TIn (float or bf16)
    const void* __restrict__ B;
    float* __restrict__ C;
    int M, N, K;
    long long sA, sB, sC;  // batch strides
    int ktiles, kt_per_split, split;
    // implicit GEMM (conv) geometry
    int H, W, Cin, P, Q, S, sh, sw, ph, pw, dh, dw;
    int vec4;    // VEC knob == 4
    int stages;  // STAGES knob
};

constexpr int cdiv_c(int a, int b) { return (a + b - 1) / b; }

template <int BM, int BN, int BK, int TT>
struct SimtCfg {
    static constexpr int NT = (BM / TT) * (BN / TT);
    static constexpr int TX = BN / TT;
    static constexpr int LDA = BM + 4;
    static constexpr int LDB = BN + 4;
    static constexpr int KV = BK / 4;                    // 4-element k groups per row
    static constexpr int SA = cdiv_c(BM * KV, NT);       // float4 staging slots per thread (A)
    static constexpr int SB = cdiv_c(BN * KV, NT);       // (B)
    static constexpr size_t SMEM = (size_t)2 * BK * (LDA + LDB) * sizeof(float) + 3 * BM * sizeof(int);
};

// compile-time half of the static validity rule (the runtime half is in sketches.cpp)
constexpr bool simt_static_ok(int BM, int BN, int BK, int TT) {
    return TT <= BM && TT <= BN && (BM / TT) * (BN / TT) <= 1024 &&
           4 * (cdiv_c(BM * (BK / 4), (BM / TT) * (BN / TT)) + cdiv_c(BN * (BK / 4), (BM / TT) * (BN / TT))) <= 64;
}

// Global loads of the input element type, widened to fp32 for the CUDA-core FMAs.
__device__ __forceinline__ float ld1(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ld1(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {  // 4 x bf16 = one 64-bit load
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xFFFF0000u));
}

// c + a * (b0, b1) as two RN fused multiply-adds in one FFMA2 (fma.rn.f32x2)
__device__ __forceinline__ float2 ffma2(float a, float b0, float b1, float2 c) {
    const float2 av = make_float2(a, a), bv = make_float2(b0, b1);
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<const unsigned long long*>(&av)), "l"(*reinterpret_cast<const unsigned long long*>(&bv)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return r;
}

// Row r of a thread's TT-row register tile -> row inside the block tile.
// TT <= 4: contiguous; TT = 8: two 4-row groups BM/2 apart (conflict-free LDS.128).
template <int BMN, int TT>
__device__ __forceinline__ int tile_row(int t, int i) {
    if constexpr (TT <= 4) return t * TT + i;
    else return (i < 4) ? (t * 4 + i) : (BMN / 2 + t * 4 + (i - 4));
}

// (r, s, c) of reduction index kk for the implicit GEMM, by carrying from a base.
struct RSC {
    int r, s, c;
};
__device__ __forceinline__ RSC rsc_advance(RSC b, int add, int Cin, int S) {
    b.c += add;
    while (b.c >= Cin) {
        b.c -= Cin;
        if (++b.s == S) { b.s = 0; ++b.r; }
    }
    return b;
}

template <int BM, int BN, int BK, int TT, int UNROLL, bool CONV, typename TIn>
__global__ void __launch_bounds__(SimtCfg<BM, BN, BK, TT>::NT)
    simt_gemm_f32_kernel(const SimtParams p) {
    using Cfg = SimtCfg<BM, BN, BK, TT>;
    constexpr int NT = Cfg::NT, TX = Cfg::TX, LDA = Cfg::LDA, LDB = Cfg::LDB, KV = Cfg::KV;
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                              // [2][BK][LDA]
    float* Bs = smem + 2 * BK * LDA;               // [2][BK][LDB]
    int* rowinfo = (int*)(Bs + 2 * BK * LDB);      // CONV: [3][BM] image base, h0, w0

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const int bz = blockIdx.z / p.split;
    const int kz = blockIdx.z % p.split;
    const int kt_begin = kz * p.kt_per_split;
    const int kt_end = min(p.ktiles, kt_begin + p.kt_per_split);
    // programmatic dependent launch: the next kernel in the stream may start its own prologue now
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (kt_begin >= kt_end) return;

    const TIn* __restrict__ A = (const TIn*)p.A + (CONV ? 0 : bz * p.sA);
    const TIn* __restrict__ B = (const TIn*)p.B + bz * p.sB;
    float* __restrict__ C = p.C + bz * p.sC;

    if constexpr (CONV) {
        for (int i = tid; i < BM; i += NT) {
            int m = m0 + i;
            int base = 0, h0 = -(1 << 29), w0 = 0;
            if (m < p.M) {
                int q = m % p.Q;
                int t = m / p.Q;
                int pp = t % p.P;
                int n = t / p.P;
                base = n * p.H * p.W * p.Cin;
                h0 = pp * p.sh - p.ph;
                w0 = q * p.sw - p.pw;
            }
            rowinfo[i] = base;
            rowinfo[BM + i] = h0;
            rowinfo[2 * BM + i] = w0;
        }
        __syncthreads();
    }

    // accumulators as column pairs: one FFMA2 (fma.rn.f32x2, sm_100) updates two of them with
    // a broadcast A value -- the same two RN fused multiply-adds, half the issue slots
    float2 acc[TT][TT / 2];
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TT / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
    auto accv = [&](int i, int j) -> float { return (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x; };

    // staging registers: each slot holds 4 consecutive k of one row
    float4 ra[Cfg::SA], rb[Cfg::SB];

    // implicit GEMM: a thread's A slots keep the same rows for every k-tile, so
    // with few slots their (image base, h0, w0) live in registers, not smem
    constexpr bool ROWREG = CONV && Cfg::SA <= 4;
    constexpr int NRR = ROWREG ? Cfg::SA : 1;
    int rbase[NRR], rh0[NRR], rw0[NRR];
    if constexpr (ROWREG) {
#pragma unroll
        for (int i = 0; i < Cfg::SA; ++i) {
            const int e = tid + i * NT, row = e / KV;
            const bool in = e < BM * KV;
            rbase[i] = in ? rowinfo[row] : 0;
            rh0[i] = in ? rowinfo[BM + row] : -(1 << 29);
            rw0[i] = in ? rowinfo[2 * BM + row] : 0;
        }
    }
    auto row_base = [&](int i, int row) -> int {
        if constexpr (ROWREG) return rbase[i]; else return rowinfo[row];
    };
    auto row_h0 = [&](int i, int row) -> int {
        if constexpr (ROWREG) return rh0[i]; else return rowinfo[BM + row];
    };
    auto row_w0 = [&](int i, int row) -> int {
        if constexpr (ROWREG) return rw0[i]; else return rowinfo[2 * BM + row];
    };

    // one A element (dense or implicit GEMM), zero outside the problem
    auto a_elem = [&](int i, int row, int kk, RSC rsc) -> float {
        if (kk >= p.K) return 0.f;
        if constexpr (CONV) {
            const int h = row_h0(i, row) + rsc.r * p.dh;
            const int w = row_w0(i, row) + rsc.s * p.dw;
            if ((unsigned)h >= (unsigned)p.H || (unsigned)w >= (unsigned)p.W) return 0.f;
            return ld1(A + row_base(i, row) + (h * p.W + w) * p.Cin + rsc.c);
        } else {
            return ld1(A + (long long)(m0 + row) * p.K + kk);
        }
    };

    // (r, s, c) of the next k-tile's first reduction index: k-tiles are loaded in
    // order, so it is carried forward by BK instead of divided out per tile
    RSC knext{0, 0, 0};
    if constexpr (CONV) {
        const int k0 = kt_begin * BK, rs = k0 / p.Cin;
        knext.c = k0 - rs * p.Cin;
        knext.s = rs % p.S;
        knext.r = rs / p.S;
    }

    auto gload = [&](int kt) {
        const int k0 = kt * BK;
        const RSC base = knext;
        if constexpr (CONV) knext = rsc_advance(knext, BK, p.Cin, p.S);
#pragma unroll
        for (int i = 0; i < Cfg::SA; ++i) {
            const int e = tid + i * NT;
            const int row = e / KV, kl = (e % KV) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < BM * KV && m0 + row < p.M) {
                RSC rsc = base;
                if constexpr (CONV) rsc = rsc_advance(base, kl, p.Cin, p.S);
                const int kk = k0 + kl;
                if (p.vec4) {  // VEC = 4: one 128-bit load (K or C is a multiple of 4)
                    if (kk < p.K) {
                        if constexpr (CONV) {
                            const int h = row_h0(i, row) + rsc.r * p.dh;
                            const int w = row_w0(i, row) + rsc.s * p.dw;
                            if ((unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W)
                                v = ld4(A + row_base(i, row) + (h * p.W + w) * p.Cin + rsc.c);
                        } else {
                            v = ld4(A + (long long)(m0 + row) * p.K + kk);
                        }
                    }
                } else {  // VEC = 1: four scalar loads
                    v.x = a_elem(i, row, kk, rsc);
                    if constexpr (CONV) rsc = rsc_advance(rsc, 1, p.Cin, p.S);
                    v.y = a_elem(i, row, kk + 1, rsc);
                    if constexpr (CONV) rsc = rsc_advance(rsc, 1, p.Cin, p.S);
                    v.z = a_elem(i, row, kk + 2, rsc);
                    if constexpr (CONV) rsc = rsc_advance(rsc, 1, p.Cin, p.S);
                    v.w = a_elem(i, row, kk + 3, rsc);
                }
            }
            ra[i] = v;
        }
#pragma unroll
        for (int i = 0; i < Cfg::SB; ++i) {
            const int e = tid + i * NT;
            const int row = e / KV, kl = (e % KV) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            const int kk = k0 + kl;
            if (e < BN * KV && n0 + row < p.N) {
                const TIn* bp = B + (long long)(n0 + row) * p.K + kk;
                if (p.vec4) {
                    if (kk < p.K) v = ld4(bp);
                } else {
                    if (kk < p.K) v.x = ld1(bp);
                    if (kk + 1 < p.K) v.y = ld1(bp + 1);
                    if (kk + 2 < p.K) v.z = ld1(bp + 2);
                    if (kk + 3 < p.K) v.w = ld1(bp + 3);
                }
            }
            rb[i] = v;
        }
    };
    auto sstore = [&](int buf) {
        float* as = As + buf * BK * LDA;
        float* bs = Bs + buf * BK * LDB;
#pragma unroll
        for (int i = 0; i < Cfg::SA; ++i) {
            const int e = tid + i * NT;
            if (e < BM * KV) {
                const int row = e / KV, kl = (e % KV) * 4;
                as[(kl + 0) * LDA + row] = ra[i].x;
                as[(kl + 1) * LDA + row] = ra[i].y;
                as[(kl + 2) * LDA + row] = ra[i].z;
                as[(kl + 3) * LDA + row] = ra[i].w;
            }
        }
#pragma unroll
        for (int i = 0; i < Cfg::SB; ++i) {
            const int e = tid + i * NT;
            if (e < BN * KV) {
                const int row = e / KV, kl = (e % KV) * 4;
                bs[(kl + 0) * LDB + row] = rb[i].x;
                bs[(kl + 1) * LDB + row] = rb[i].y;
                bs[(kl + 2) * LDB + row] = rb[i].z;
                bs[(kl + 3) * LDB + row] = rb[i].w;
            }
        }
    };
    auto compute = [&](int buf) {
        const float* as = As + buf * BK * LDA;
        const float* bs = Bs + buf * BK * LDB;
#pragma unroll UNROLL
        for (int k = 0; k < BK; ++k) {
            float a[TT], b[TT];
            if constexpr (TT == 2) {
                float2 va = *reinterpret_cast<const float2*>(as + k * LDA + ty * 2);
                float2 vb = *reinterpret_cast<const float2*>(bs + k * LDB + tx * 2);
                a[0] = va.x; a[1] = va.y; b[0] = vb.x; b[1] = vb.y;
            } else {
#pragma unroll
                for (int g = 0; g < TT / 4; ++g) {
                    float4 va = *reinterpret_cast<const float4*>(as + k * LDA + tile_row<BM, TT>(ty, 4 * g));
                    float4 vb = *reinterpret_cast<const float4*>(bs + k * LDB + tile_row<BN, TT>(tx, 4 * g));
                    a[4 * g + 0] = va.x; a[4 * g + 1] = va.y; a[4 * g + 2] = va.z; a[4 * g + 3] = va.w;
                    b[4 * g + 0] = vb.x; b[4 * g + 1] = vb.y; b[4 * g + 2] = vb.z; b[4 * g + 3] = vb.w;
                }
            }
#pragma unroll
            for (int i = 0; i < TT; ++i)
#pragma unroll
                for (int j = 0; j < TT / 2; ++j) acc[i][j] = ffma2(a[i], b[2 * j], b[2 * j + 1], acc[i][j]);
        }
    };

    // launched with programmatic stream serialization: the prologue above overlaps the preceding
    // kernel's tail; X and W are read only after it completed -- except behind this schedule's own
    // split-K zeroing kernel, which is plainly serialised (every earlier kernel is complete when it
    // starts), so the wait is deferred to the first atomic (Y zeroed)
    if (p.split == 1) griddep_wait();
    if (p.stages >= 2) {  // STAGES = 2: register prefetch of the next tile overlaps the FMAs
        gload(kt_begin);
        sstore(0);
        __syncthreads();
        int buf = 0;
        for (int kt = kt_begin; kt < kt_end; ++kt) {
            const bool more = kt + 1 < kt_end;
            if (more) gload(kt + 1);
            compute(buf);
            if (more) {
                sstore(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    } else {  // STAGES = 1: load, sync, compute, sync
        for (int kt = kt_begin; kt < kt_end; ++kt) {
            gload(kt);
            sstore(0);
            __syncthreads();
            compute(0);
            __syncthreads();
        }
    }

    // epilogue: direct stores (SPLIT_K = 1) or atomic partial-sum reduction
    const bool atomic = p.split > 1;
    if (atomic) griddep_wait();  // Y zeroed by the prerequisite grid (PDL)
#pragma unroll
    for (int i = 0; i < TT; ++i) {
        const int m = m0 + tile_row<BM, TT>(ty, i);
        if (m >= p.M) continue;
        float* crow = C + (long long)m * p.N;
#pragma unroll
        for (int g = 0; g < (TT + 3) / 4; ++g) {
            constexpr int W = TT < 4 ? TT : 4;
            const int n = n0 + tile_row<BN, TT>(tx, W * g);
            if (W == 4 && n + 3 < p.N && (p.N % 4) == 0) {
                float4 v = make_float4(accv(i, 4 * g), accv(i, 4 * g + 1), accv(i, 4 * g + 2), accv(i, 4 * g + 3));
                if (atomic) atomicAdd(reinterpret_cast<float4*>(crow + n), v);
                else *reinterpret_cast<float4*>(crow + n) = v;
            } else if (W == 2 && n + 1 < p.N && (p.N % 2) == 0) {
                float2 v = make_float2(accv(i, 0), accv(i, 1));
                if (atomic) atomicAdd(reinterpret_cast<float2*>(crow + n), v);
                else *reinterpret_cast<float2*>(crow + n) = v;
            } else {
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    if (n + j < p.N) {
                        if (atomic) atomicAdd(crow + n + j, accv(i, W * g + j));
                        else crow[n + j] = accv(i, W * g + j);
                    }
                }
            }
        }
    }
}

template <int BM, int BN, int BK, int TT, int UNROLL, bool CONV, typename TIn = float>
cudaError_t simt_launch(const LaunchCtx& c) {
    using Cfg = SimtCfg<BM, BN, BK, TT>;
    auto kern = simt_gemm_f32_kernel<BM, BN, BK, TT, UNROLL, CONV, TIn>;
    static std::atomic<unsigned long long> optin{0};
    {
        cudaError_t e = smem_optin(optin, kern, (int)Cfg::SMEM);
        if (e != cudaSuccess) return e;
    }
    const ShapeInfo& s = *c.sh;
    SimtParams p;
    p.A = c.x;
    p.B = c.w;
    p.C = (float*)c.y;
    p.M = (int)s.M; p.N = (int)s.N; p.K = (int)s.K;
    p.sA = s.M * s.K; p.sB = s.N * s.K; p.sC = s.M * s.N;
    p.ktiles = (int)((s.K + BK - 1) / BK);
    p.split = c.split;
    p.kt_per_split = (p.ktiles + c.split - 1) / c.split;
    p.H = (int)s.h; p.W = (int)s.w; p.Cin = (int)s.c; p.P = (int)s.p; p.Q = (int)s.q; p.S = (int)s.s;
    p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
    p.vec4 = c.vec == 4;
    p.stages = c.stages;
    if (c.split > 1) {
        cudaError_t e = zero_for_splitk((float*)c.y, s.y_elems, c.stream);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((s.M + BM - 1) / BM), (unsigned)((s.N + BN - 1) / BN), (unsigned)(s.batch * c.split));
    cfg.blockDim = dim3(Cfg::NT);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];  // always a programmatic dependent launch (see the kernel)
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    count_launches(1);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int BM, int BN, int BK, int TT, int UNROLL, bool CONV>
void simt_register() {
    if constexpr (simt_static_ok(BM, BN, BK, TT)) {
        registry_add(kernel_key(CONV ? SK_SIMT_IGEMM_CONV_F32 : SK_SIMT_GEMM_F32, BM, BN, BK, TT, UNROLL),
                     &simt_launch<BM, BN, BK, TT, UNROLL, CONV>);
    }
}

// bf16 inputs (CUDA-core FMAs on widened values, fp32 accumulate): implicit-GEMM conv only
template <int BM, int BN, int BK, int TT, int UNROLL>
void simt_register_bf16() {
    if constexpr (simt_static_ok(BM, BN, BK, TT)) {
        registry_add(kernel_key(SK_SIMT_IGEMM_CONV_BF16, BM, BN, BK, TT, UNROLL),
                     &simt_launch<BM, BN, BK, TT, UNROLL, true, __nv_bfloat16>);
    }
}

}  // namespace db200
