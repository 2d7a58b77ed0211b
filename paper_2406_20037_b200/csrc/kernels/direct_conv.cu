// direct_conv.cu — sketches SIMT_DIRECT_CONV_F32 / SIMT_DIRECT_CONV_BF16 (SURVEY §8(d).1's
// `simt_direct_conv` template): the conv2d loop nest of Def. 2.1 without the GEMM
// view, for layers with few input channels (C <= 16: the RGB stems of VGG / AlexNet / ResNet),
// where an implicit GEMM has a reduction of only C*R*S = 27..363 and its gathers dominate.
//
// Schedule: a CTA owns PX*TP consecutive output pixels (NPQ order) x BKC output channels; the
// CTA's filters are staged once in shared memory as [R*S*C][BKC] fp32; each thread owns TP
// pixels (PX apart, so a warp's lanes stay on consecutive pixels) and KT consecutive channels,
// walks the taps (r, s, c) reading each input element once (zero outside the image) and updates
// TP x KT accumulators with FFMA2 (broadcast input value x pairs of filter values; each float4
// filter broadcast -- every lane of a warp shares its channel group -- feeds 2*TP FFMA2).
// Epilogue: EPI 0 = each thread stores its KT channels per pixel (float4); EPI 1 = the tile is
// staged through shared memory and written as contiguous rows.
// Annotations: KT, TP (compile-time), PX, BKC, EPI (runtime).  fp32 accumulation, fp32 output.
#include <cuda_bf16.h>

#include "common.cuh"

namespace db200 {

struct DirectParams {
    const void* __restrict__ X;
    const void* __restrict__ Wt;
    float* __restrict__ Y;
    int N, H, W, C, K, R, S, P, Q, sh, sw, ph, pw, dh, dw;
    int M;  // N * P * Q
    int px, bkc, epi;
};

__device__ __forceinline__ float dld(const float* p) { return __ldg(p); }
__device__ __forceinline__ float dld(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }

__device__ __forceinline__ float2 dffma2(float a, float b0, float b1, float2 c) {
    const float2 av = make_float2(a, a), bv = make_float2(b0, b1);
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<const unsigned long long*>(&av)), "l"(*reinterpret_cast<const unsigned long long*>(&bv)),
          "l"(*reinterpret_cast<const unsigned long long*>(&c)));
    return r;
}

template <typename TIn, int KT, int TP>
__global__ void __launch_bounds__(direct_max_threads(KT, TP)) direct_conv_kernel(const DirectParams p) {
    extern __shared__ __align__(16) float dsm[];
    const int RSC = p.R * p.S * p.C, BKC = p.bkc, PX = p.px;
    float* wsm = dsm;  // [RSC][BKC]
    const int tid = threadIdx.x;
    const int pxl = tid % PX, kg = tid / PX;
    const int m0 = blockIdx.x * PX * TP, k0 = blockIdx.y * BKC;
    const TIn* __restrict__ X = (const TIn*)p.X;
    const TIn* __restrict__ Wt = (const TIn*)p.Wt;

    // filters of this CTA's channel block, transposed to [rsc][k] (zero past K)
    for (int e = tid; e < BKC * RSC; e += blockDim.x) {
        const int k = e / RSC, j = e - k * RSC;
        wsm[j * BKC + k] = (k0 + k < p.K) ? dld(Wt + (long long)(k0 + k) * RSC + j) : 0.f;
    }
    __syncthreads();

    bool live[TP];
    int nb[TP], h0[TP], w0[TP];
    bool any = false;
#pragma unroll
    for (int u = 0; u < TP; ++u) {
        const int m = m0 + pxl + u * PX;
        live[u] = m < p.M;
        any |= live[u];
        nb[u] = 0; h0[u] = -(1 << 29); w0[u] = 0;  // a dead pixel reads nothing (h out of range)
        if (live[u]) {
            const int q = m % p.Q, t = m / p.Q, pp = t % p.P;
            nb[u] = (t / p.P) * p.H;
            h0[u] = pp * p.sh - p.ph;
            w0[u] = q * p.sw - p.pw;
        }
    }
    float2 acc[TP][KT / 2];
#pragma unroll
    for (int u = 0; u < TP; ++u)
#pragma unroll
        for (int j = 0; j < KT / 2; ++j) acc[u][j] = make_float2(0.f, 0.f);
    const float* wk = wsm + kg * KT;
    if (any) {
        for (int r = 0; r < p.R; ++r) {
            for (int s = 0; s < p.S; ++s) {
                bool ok[TP];
                const TIn* xp[TP];
#pragma unroll
                for (int u = 0; u < TP; ++u) {
                    const int h = h0[u] + r * p.dh, w = w0[u] + s * p.dw;
                    ok[u] = (unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W;
                    xp[u] = X + ((long long)(nb[u] + (ok[u] ? h : 0)) * p.W + (ok[u] ? w : 0)) * p.C;
                }
                const float* wr = wk + (r * p.S + s) * p.C * BKC;
                for (int c = 0; c < p.C; ++c) {
                    float x[TP];
#pragma unroll
                    for (int u = 0; u < TP; ++u) x[u] = ok[u] ? dld(xp[u] + c) : 0.f;
                    const float* wc = wr + c * BKC;
#pragma unroll
                    for (int j = 0; j < KT / 4; ++j) {
                        const float4 w4 = *reinterpret_cast<const float4*>(wc + 4 * j);
#pragma unroll
                        for (int u = 0; u < TP; ++u) {
                            acc[u][2 * j] = dffma2(x[u], w4.x, w4.y, acc[u][2 * j]);
                            acc[u][2 * j + 1] = dffma2(x[u], w4.z, w4.w, acc[u][2 * j + 1]);
                        }
                    }
                }
            }
        }
    }

    const int kb = k0 + kg * KT;  // this thread's first channel
    if (p.epi == 0) {
        const bool vec = (p.K % 4) == 0;
#pragma unroll
        for (int u = 0; u < TP; ++u) {
            if (!live[u]) continue;
            float* yp = p.Y + (long long)(m0 + pxl + u * PX) * p.K + kb;
#pragma unroll
            for (int j = 0; j < KT / 4; ++j) {
                const float4 v = make_float4(acc[u][2 * j].x, acc[u][2 * j].y, acc[u][2 * j + 1].x, acc[u][2 * j + 1].y);
                if (vec && kb + 4 * j + 3 < p.K) {
                    *reinterpret_cast<float4*>(yp + 4 * j) = v;
                } else {
                    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (kb + 4 * j + e < p.K) yp[4 * j + e] = vv[e];
                }
            }
        }
        return;
    }
    // EPI 1: the tile through shared memory ([PX * TP][BKC + 4]), then contiguous row stores
    __syncthreads();  // filters no longer needed: the staging tile reuses their space
    const int LD = BKC + 4;
    float* ysm = dsm;
#pragma unroll
    for (int u = 0; u < TP; ++u)
#pragma unroll
        for (int j = 0; j < KT / 4; ++j)
            *reinterpret_cast<float4*>(ysm + (pxl + u * PX) * LD + kg * KT + 4 * j) =
                make_float4(acc[u][2 * j].x, acc[u][2 * j].y, acc[u][2 * j + 1].x, acc[u][2 * j + 1].y);
    __syncthreads();
    const int c4 = BKC / 4;
    const bool vec = (p.K % 4) == 0;
    for (int e = tid; e < PX * TP * c4; e += blockDim.x) {
        const int row = e / c4, col = (e - row * c4) * 4;
        const int mm = m0 + row, kk = k0 + col;
        if (mm >= p.M || kk >= p.K) continue;
        const float4 v = *reinterpret_cast<const float4*>(ysm + row * LD + col);
        float* yp = p.Y + (long long)mm * p.K + kk;
        if (vec && kk + 3 < p.K) {
            *reinterpret_cast<float4*>(yp) = v;
        } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
            for (int u = 0; u < 4; ++u)
                if (kk + u < p.K) yp[u] = vv[u];
        }
    }
}

template <typename TIn, int KT, int TP>
cudaError_t direct_launch(const LaunchCtx& c) {
    auto kern = direct_conv_kernel<TIn, KT, TP>;
    static std::atomic<unsigned long long> optin{0};
    {
        cudaError_t e = smem_optin(optin, kern, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const ShapeInfo& s = *c.sh;
    DirectParams p;
    p.X = c.x; p.Wt = c.w; p.Y = (float*)c.y;
    p.N = (int)s.n; p.H = (int)s.h; p.W = (int)s.w; p.C = (int)s.c; p.K = (int)s.k; p.R = (int)s.r; p.S = (int)s.s;
    p.P = (int)s.p; p.Q = (int)s.q; p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
    p.M = (int)s.M;
    p.px = c.dims[0]; p.bkc = c.dims[1]; p.epi = c.dims[2];
    const size_t smem = direct_smem_bytes((int)(s.r * s.s * s.c), p.bkc, p.px * TP, p.epi);
    dim3 grid((unsigned)((s.M + p.px * TP - 1) / (p.px * TP)), (unsigned)((s.k + p.bkc - 1) / p.bkc));
    kern<<<grid, (unsigned)(p.px * (p.bkc / KT)), smem, c.stream>>>(p);
    count_launches(1);
    return cudaGetLastError();
}

template <int KT, int TP>
void direct_register() {
    if constexpr (KT * TP <= 64) {  // accumulators per thread (register budget; the validity rule)
        registry_add(kernel_key(SK_SIMT_DIRECT_CONV_F32, KT, TP, 0, 0, 0), &direct_launch<float, KT, TP>);
        registry_add(kernel_key(SK_SIMT_DIRECT_CONV_BF16, KT, TP, 0, 0, 0), &direct_launch<__nv_bfloat16, KT, TP>);
    }
}
template <int KT>
void direct_register_tp() {
    direct_register<KT, 1>();
    direct_register<KT, 2>();
    direct_register<KT, 4>();
}

void register_direct_conv() {
    direct_register_tp<4>();
    direct_register_tp<8>();
    direct_register_tp<16>();
    direct_register_tp<32>();
    direct_register_tp<64>();
}

}  // namespace db200
