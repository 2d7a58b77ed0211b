// tc_gemm.cu — sketch TC_GEMM_BF16: dense / batch_matmul on the 5th-generation
// tensor cores.  Y[b,m,n] (fp32) = sum_k X[b,m,k] W[b,n,k], X and W bf16.
//
// The sketch (Def. 2.1): tile (m, n) into 128 x BN output tiles, one CTA each
// (x SPLIT_K slices of the k range); stage BK-wide k slices of A and B through
// a STAGES-deep shared-memory ring filled by TMA (128-byte swizzle, one
// mbarrier pair per stage); accumulate in TMEM with tcgen05.mma issued by a
// single thread (UMMA 128 x BN x 16); drain TMEM with tcgen05.ld in four
// epilogue warps straight to global memory (fp32), or with vector reductions
// (red.global.add.v4.f32) into a zeroed Y when SPLIT_K > 1.
// Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
// Knobs: BM (128), BN, BK, STAGES, SPLIT_K.
#include <cstring>

#include "common.cuh"
#include "tc_common.cuh"

namespace db200 {

template <int BN, int BK, int STAGES>
struct TcCfg {
    static constexpr int BM = 128;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
    static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
    static constexpr int THREADS = 192;
};

struct TcParams {
    int M, N, K;
    int kblocks, kb_per_split, split;
    float* C;
    long long sC;
};

template <int BN, int BK, int STAGES>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const TcParams p) {
    using Cfg = TcCfg<BN, BK, STAGES>;
    constexpr int BM = Cfg::BM;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + STAGES * Cfg::STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tmem_full = bars + 2 * STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int bz = blockIdx.z / p.split, kz = blockIdx.z % p.split;
    const int kb0 = kz * p.kb_per_split;
    const int kb1 = min(p.kblocks, kb0 + p.kb_per_split);
    const int nkb = kb1 - kb0;
    if (nkb <= 0) return;  // uniform per CTA, before any barrier

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(tc::smem_u32(&full[s]), 1);
            tc::mbar_init(tc::smem_u32(&empty[s]), 1);
        }
        tc::mbar_init(tc::smem_u32(tmem_full), 1);
        tc::fence_barrier_init();
        tc::tma_prefetch(&tmA);
        tc::tma_prefetch(&tmB);
    }
    if (warp == 1) tc::tmem_alloc<Cfg::TMEM_COLS>(tc::smem_u32(tmem_slot));
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
                tc::mbar_wait(tc::smem_u32(&empty[s]), ph ^ 1u);
                const uint32_t fb = tc::smem_u32(&full[s]);
                tc::mbar_expect_tx(fb, Cfg::STAGE_BYTES);
                const int k0 = (kb0 + i) * BK;
                const uint32_t sa = tc::smem_u32(base + s * Cfg::STAGE_BYTES);
                const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
                for (int a = 0; a < BK / 64; ++a) {
                    tc::tma_load_3d(sa + a * BM * 128, &tmA, fb, k0 + a * 64, m0, bz);
                    tc::tma_load_3d(sb + a * BN * 128, &tmB, fb, k0 + a * 64, n0, bz);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = tc::idesc_bf16(BM, BN);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
                tc::mbar_wait(tc::smem_u32(&full[s]), ph);
                tc::tc_fence_after();
                const uint32_t sa = tc::smem_u32(base + s * Cfg::STAGE_BYTES);
                const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint32_t atom = k / 4, inner = (k % 4) * 32;
                    const uint64_t da = tc::sdesc_sw128(sa + atom * BM * 128 + inner);
                    const uint64_t db = tc::sdesc_sw128(sb + atom * BN * 128 + inner);
                    tc::umma_bf16(tmem, da, db, idesc, (i > 0 || k > 0) ? 1u : 0u);
                }
                tc::umma_commit(tc::smem_u32(&empty[s]));  // frees the stage when these MMAs finish
            }
            tc::umma_commit(tc::smem_u32(tmem_full));
        }
    } else {  // ---- epilogue: TMEM -> registers -> global
        const int q = warp & 3;
        const int row = m0 + q * 32 + lane;
        tc::mbar_wait(tc::smem_u32(tmem_full), 0);
        tc::tc_fence_after();
        float* crow = p.C + bz * p.sC + (long long)row * p.N;
        const bool vec_ok = (p.N % 4) == 0;
#pragma unroll 1
        for (int c = 0; c < BN / 16; ++c) {
            uint32_t r[16];
            tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 16), r);
            tc::tmem_ld_wait();
            const int n = n0 + c * 16;
            if (row >= p.M || n >= p.N) continue;
            if (vec_ok && n + 16 <= p.N) {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    float4 f = make_float4(__uint_as_float(r[4 * v]), __uint_as_float(r[4 * v + 1]),
                                           __uint_as_float(r[4 * v + 2]), __uint_as_float(r[4 * v + 3]));
                    if (p.split > 1) tc::red_add_v4(crow + n + 4 * v, f.x, f.y, f.z, f.w);
                    else *reinterpret_cast<float4*>(crow + n + 4 * v) = f;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (n + j < p.N) {
                        if (p.split > 1) atomicAdd(crow + n + j, __uint_as_float(r[j]));
                        else crow[n + j] = __uint_as_float(r[j]);
                    }
                }
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem);
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

// 3-D K-major bf16 operand [batch][rows][K] -> box {64, box_rows, 1}, 128-byte swizzle
static bool make_kmajor_map(CUtensorMap* m, const void* ptr, int64_t batch, int64_t rows, int64_t K, int box_rows) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)(rows * K * 2)};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN, int BK, int STAGES>
cudaError_t tc_gemm_launch(const LaunchCtx& c) {
    using Cfg = TcCfg<BN, BK, STAGES>;
    auto kern = tc_gemm_bf16_kernel<BN, BK, STAGES>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    const ShapeInfo& s = *c.sh;
    CUtensorMap ta, tb;
    if (!make_kmajor_map(&ta, c.x, s.batch, s.M, s.K, Cfg::BM) || !make_kmajor_map(&tb, c.w, s.batch, s.N, s.K, BN))
        return cudaErrorInvalidValue;
    TcParams p;
    p.M = (int)s.M; p.N = (int)s.N; p.K = (int)s.K;
    p.kblocks = (int)((s.K + BK - 1) / BK);
    p.split = c.split;
    p.kb_per_split = (p.kblocks + c.split - 1) / c.split;
    p.C = (float*)c.y;
    p.sC = s.M * s.N;
    if (c.split > 1) {
        cudaError_t e = cudaMemsetAsync(c.y, 0, (size_t)s.y_elems * sizeof(float), c.stream);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((unsigned)((s.M + Cfg::BM - 1) / Cfg::BM), (unsigned)((s.N + BN - 1) / BN),
              (unsigned)(s.batch * c.split));
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, c.stream>>>(ta, tb, p);
    count_launches(1);
    return cudaGetLastError();
}

constexpr bool tc_static_ok(int BN, int BK, int STAGES) {
    return 1024 + (size_t)STAGES * (128 + BN) * BK * 2 + 256 <= 227 * 1024;
}

template <int BN, int BK, int STAGES>
void tc_register() {
    if constexpr (tc_static_ok(BN, BK, STAGES))
        registry_add(kernel_key(SK_TC_GEMM_BF16, 128, BN, BK, STAGES, 0), &tc_gemm_launch<BN, BK, STAGES>);
}

#define TC_STAGES(BN, BK) \
    tc_register<BN, BK, 2>(); tc_register<BN, BK, 3>(); tc_register<BN, BK, 4>(); tc_register<BN, BK, 6>();

void register_tc_gemm() {
    TC_STAGES(64, 64) TC_STAGES(128, 64) TC_STAGES(256, 64)
    TC_STAGES(64, 128) TC_STAGES(128, 128) TC_STAGES(256, 128)
}

}  // namespace db200
