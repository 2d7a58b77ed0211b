// dwconv.cu — sketches SIMT_DWCONV_F32 and SIMT_DWCONV_BF16.
//
// Depthwise conv2d (groups = C = K, R-C5): Y[n,p,q,c] = sum_{r,s} X[n, p*sh-ph+r*dh,
// q*sw-pw+s*dw, c] * W[c,r,s].  Each output reads R*S inputs of ONE channel, so the
// op has no reduction over channels and no tensor-core shape: it is bound by HBM
// (|X| + |W| + |Y| once) or, at batch 1, by latency.  The schedule therefore works
// on coalescing, reuse and instruction count, not on a GEMM view:
//   - channels are the fastest NHWC dimension: VEC consecutive channels per thread
//     (one 32/64/128-bit load per tap), CT threads across channels;
//   - QT x PT threads across output columns / rows, TQ consecutive output columns
//     and TP consecutive output rows per thread;
//   - ALG 0 (register window): filter taps in registers, the thread walks the input
//     rows its TP x TQ outputs need and loads each row segment ONCE into registers
//     (every input vector feeds up to TP x TQ outputs); R = S and the stride are
//     compile-time (3x3 / 5x5, stride 1 / 2: every depthwise layer of the sweep);
//     no shared memory, no barrier;
//   - ALG 1 stages the CTA's input window (output tile + halo) in shared memory
//     once, converted to fp32; ALG 2 reads every tap through L1 (__ldg); both keep
//     the CTA's filters transposed to [r*S+s][channel] in shared memory and take
//     any R, S, stride and dilation (TP = 1).
// Knobs: VEC, TQ, TP, ALG compile-time; CT, QT, PT runtime (the thread-block shape).
// fp32 FMAs on the CUDA cores; bf16 inputs are widened at load, fp32 accumulate/out.
#include <cuda_bf16.h>

#include "common.cuh"

namespace db200 {

struct DwParams {
    const void* __restrict__ x;
    const void* __restrict__ w;
    float* __restrict__ y;
    int N, H, W, C, R, S, P, Q, sh, sw, ph, pw, dh, dw;
    int tiles_p;  // ceil(P / PT)
    int ih, iw;   // SMEM input window: rows, columns
};

template <typename T, int VEC>
struct Vec;
template <>
struct Vec<float, 1> {
    static __device__ __forceinline__ void load(const float* p, float* o) { o[0] = __ldg(p); }
};
template <>
struct Vec<float, 2> {
    static __device__ __forceinline__ void load(const float* p, float* o) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = v.x; o[1] = v.y;
    }
};
template <>
struct Vec<float, 4> {
    static __device__ __forceinline__ void load(const float* p, float* o) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};
__device__ __forceinline__ float bf_lo(unsigned u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(unsigned u) { return __uint_as_float(u & 0xFFFF0000u); }
template <>
struct Vec<__nv_bfloat16, 1> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* o) { o[0] = __bfloat162float(__ldg(p)); }
};
template <>
struct Vec<__nv_bfloat16, 2> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* o) {
        const unsigned u = __ldg(reinterpret_cast<const unsigned*>(p));
        o[0] = bf_lo(u); o[1] = bf_hi(u);
    }
};
template <>
struct Vec<__nv_bfloat16, 4> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* o) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        o[0] = bf_lo(u.x); o[1] = bf_hi(u.x); o[2] = bf_lo(u.y); o[3] = bf_hi(u.y);
    }
};
template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <int VEC>
__device__ __forceinline__ void store_vec(float* p, const float* v) {
    if constexpr (VEC == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else if constexpr (VEC == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    else p[0] = v[0];
}

template <typename TIn, int VEC, int TQ, bool SMEM>
__global__ void __launch_bounds__(512) dwconv_kernel(const DwParams p) {
    extern __shared__ __align__(16) float sm[];
    const int ct = blockDim.x, qt = blockDim.y, pt = blockDim.z;
    const int ctv = ct * VEC;  // channels per CTA
    const int tid = threadIdx.x + ct * (threadIdx.y + qt * threadIdx.z);
    const int nthr = ct * qt * pt;
    const int c_cta = blockIdx.x * ctv;
    const int q_cta = blockIdx.y * qt * TQ;
    const int n = blockIdx.z / p.tiles_p;
    const int p_cta = (blockIdx.z % p.tiles_p) * pt;
    const int RS = p.R * p.S;
    const TIn* __restrict__ X = (const TIn*)p.x;
    const TIn* __restrict__ Wt = (const TIn*)p.w;
    // programmatic dependent launch: the next kernel may launch now; this one reads only after its
    // predecessor completed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    griddep_wait();

    // filters of this CTA's channels, transposed to [rs][channel] (zero past C)
    float* ws = sm;
    for (int i = tid; i < RS * ctv; i += nthr) {
        const int rs = i / ctv, cl = i - rs * ctv, c = c_cta + cl;
        ws[i] = c < p.C ? to_f32(Wt[(long long)c * RS + rs]) : 0.f;
    }
    float* xs = ws + RS * ctv;  // SMEM: [ih][iw][ctv]
    const int h0 = p_cta * p.sh - p.ph, w0 = q_cta * p.sw - p.pw;
    const long long img = (long long)n * p.H * p.W * p.C;
    if constexpr (SMEM) {
        const int cvs = ct;  // VEC-wide channel groups per window position
        const int total = p.ih * p.iw * cvs;
        for (int i = tid; i < total; i += nthr) {
            const int cv = i % cvs, pos = i / cvs;
            const int col = pos % p.iw, row = pos / p.iw;
            const int h = h0 + row, w = w0 + col, c = c_cta + cv * VEC;
            float v[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) v[e] = 0.f;
            if ((unsigned)h < (unsigned)p.H && (unsigned)w < (unsigned)p.W && c < p.C)
                Vec<TIn, VEC>::load(X + img + ((long long)h * p.W + w) * p.C + c, v);
            float* d = xs + (size_t)pos * ctv + cv * VEC;
#pragma unroll
            for (int e = 0; e < VEC; ++e) d[e] = v[e];
        }
    }
    __syncthreads();

    const int cl = threadIdx.x * VEC;  // channel offset inside the CTA
    const int c = c_cta + cl;
    const int pp = p_cta + threadIdx.z;
    const int q0 = q_cta + threadIdx.y * TQ;
    if (c >= p.C || pp >= p.P || q0 >= p.Q) return;

    float acc[TQ][VEC];
#pragma unroll
    for (int t = 0; t < TQ; ++t)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[t][e] = 0.f;

    for (int r = 0; r < p.R; ++r) {
        const int hr = threadIdx.z * p.sh + r * p.dh;  // window row (SMEM) / offset from h0
        const int h = h0 + hr;
        if (!SMEM && (unsigned)h >= (unsigned)p.H) continue;
        for (int s = 0; s < p.S; ++s) {
            float wv[VEC];
            const float* wp = ws + (r * p.S + s) * ctv + cl;
#pragma unroll
            for (int e = 0; e < VEC; ++e) wv[e] = wp[e];
#pragma unroll
            for (int t = 0; t < TQ; ++t) {
                const int wc = (threadIdx.y * TQ + t) * p.sw + s * p.dw;  // window column
                float xv[VEC];
                if constexpr (SMEM) {
                    const float* xp = xs + ((size_t)hr * p.iw + wc) * ctv + cl;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) xv[e] = xp[e];
                } else {
                    const int w = w0 + wc;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) xv[e] = 0.f;
                    if ((unsigned)w < (unsigned)p.W) Vec<TIn, VEC>::load(X + img + ((long long)h * p.W + w) * p.C + c, xv);
                }
#pragma unroll
                for (int e = 0; e < VEC; ++e) acc[t][e] = fmaf(xv[e], wv[e], acc[t][e]);
            }
        }
    }
    float* yrow = p.y + (((long long)n * p.P + pp) * p.Q) * p.C + c;
#pragma unroll
    for (int t = 0; t < TQ; ++t)
        if (q0 + t < p.Q) store_vec<VEC>(yrow + (long long)(q0 + t) * p.C, acc[t]);
}

// ALG 0: register window.  Compile-time KS = R = S and SH = sh = sw (dilation 1).
template <typename TIn, int VEC, int TQ, int TP, int KS, int SH>
__global__ void __launch_bounds__(512) dwconv_win_kernel(const DwParams p) {
    constexpr int NR = (TP - 1) * SH + KS;  // input rows behind TP output rows
    constexpr int NC = (TQ - 1) * SH + KS;  // input columns behind TQ output columns
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * VEC;
    const int q0 = (blockIdx.y * blockDim.y + threadIdx.y) * TQ;
    const int n = blockIdx.z / p.tiles_p;
    const int p0 = ((blockIdx.z % p.tiles_p) * blockDim.z + threadIdx.z) * TP;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // PDL, as dwconv_kernel
    if (c >= p.C || q0 >= p.Q || p0 >= p.P) return;
    griddep_wait();
    const TIn* __restrict__ X = (const TIn*)p.x + (long long)n * p.H * p.W * p.C + c;
    const TIn* __restrict__ Wt = (const TIn*)p.w + (long long)c * KS * KS;

    float wr[KS * KS][VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e)
#pragma unroll
        for (int rs = 0; rs < KS * KS; ++rs) wr[rs][e] = to_f32(__ldg(Wt + e * KS * KS + rs));
    float acc[TP][TQ][VEC];
#pragma unroll
    for (int a = 0; a < TP; ++a)
#pragma unroll
        for (int b = 0; b < TQ; ++b)
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[a][b][e] = 0.f;

    const int h0 = p0 * SH - p.ph, w0 = q0 * SH - p.pw;
    // column offsets and bounds are the same for every input row
    int coff[NC];
    bool cok[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        coff[j] = (w0 + j) * p.C;
        cok[j] = (unsigned)(w0 + j) < (unsigned)p.W;
    }
    // two input rows in flight: row i + 1 is loaded while row i feeds the FMAs
    float xr[2][NC][VEC];
    auto load_row = [&](int i, float (&dst)[NC][VEC]) {
        const int h = h0 + i;
        const bool hok = (unsigned)h < (unsigned)p.H;
        const TIn* rowp = X + (long long)h * p.W * p.C;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) dst[j][e] = 0.f;
            if (hok && cok[j]) Vec<TIn, VEC>::load(rowp + coff[j], dst[j]);
        }
    };
    load_row(0, xr[0]);
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        if (i + 1 < NR) load_row(i + 1, xr[(i + 1) & 1]);
        const float(&cur)[NC][VEC] = xr[i & 1];
#pragma unroll
        for (int a = 0; a < TP; ++a) {
            const int r = i - a * SH;  // compile-time after unrolling
            if (r < 0 || r >= KS) continue;
#pragma unroll
            for (int b = 0; b < TQ; ++b)
#pragma unroll
                for (int s = 0; s < KS; ++s)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) acc[a][b][e] = fmaf(cur[b * SH + s][e], wr[r * KS + s][e], acc[a][b][e]);
        }
    }
#pragma unroll
    for (int a = 0; a < TP; ++a) {
        if (p0 + a >= p.P) break;
        float* yrow = p.y + (((long long)n * p.P + p0 + a) * p.Q) * p.C + c;
#pragma unroll
        for (int b = 0; b < TQ; ++b)
            if (q0 + b < p.Q) store_vec<VEC>(yrow + (long long)(q0 + b) * p.C, acc[a][b]);
    }
}

template <typename TIn, int VEC, int TQ, int TP, int KS, int SH>
cudaError_t dwconv_win_launch(const LaunchCtx& c) {
    const ShapeInfo& s = *c.sh;
    const int ct = c.dims[0], qt = c.dims[1], pt = c.dims[2];
    DwParams p;
    p.x = c.x;
    p.w = c.w;
    p.y = (float*)c.y;
    p.N = (int)s.n; p.H = (int)s.h; p.W = (int)s.w; p.C = (int)s.c; p.R = (int)s.r; p.S = (int)s.s;
    p.P = (int)s.p; p.Q = (int)s.q;
    p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
    p.tiles_p = (p.P + pt * TP - 1) / (pt * TP);
    p.ih = p.iw = 0;
    dim3 grid((unsigned)((p.C + ct * VEC - 1) / (ct * VEC)), (unsigned)((p.Q + qt * TQ - 1) / (qt * TQ)),
              (unsigned)(p.N * p.tiles_p));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(ct, qt, pt);
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, dwconv_win_kernel<TIn, VEC, TQ, TP, KS, SH>, p);
    count_launches(1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename TIn, int VEC, int TQ, bool SMEM>
cudaError_t dwconv_launch(const LaunchCtx& c) {
    auto kern = dwconv_kernel<TIn, VEC, TQ, SMEM>;
    static std::atomic<unsigned long long> optin{0};
    {
        cudaError_t e = smem_optin(optin, kern, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    const ShapeInfo& s = *c.sh;
    const int ct = c.dims[0], qt = c.dims[1], pt = c.dims[2];
    DwParams p;
    p.x = c.x;
    p.w = c.w;
    p.y = (float*)c.y;
    p.N = (int)s.n; p.H = (int)s.h; p.W = (int)s.w; p.C = (int)s.c; p.R = (int)s.r; p.S = (int)s.s;
    p.P = (int)s.p; p.Q = (int)s.q;
    p.sh = s.sh; p.sw = s.sw; p.ph = s.ph; p.pw = s.pw; p.dh = s.dh; p.dw = s.dw;
    p.tiles_p = (p.P + pt - 1) / pt;
    p.ih = (pt - 1) * p.sh + (p.R - 1) * p.dh + 1;
    p.iw = (qt * TQ - 1) * p.sw + (p.S - 1) * p.dw + 1;
    const size_t smem = dwconv_smem_bytes(p.R * p.S, ct * VEC, SMEM ? p.ih * p.iw : 0);
    dim3 grid((unsigned)((p.C + ct * VEC - 1) / (ct * VEC)), (unsigned)((p.Q + qt * TQ - 1) / (qt * TQ)),
              (unsigned)(p.N * p.tiles_p));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(ct, qt, pt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute attr[1];
    pdl_attr(attr[0]);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    count_launches(1);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// registry key: (VEC, TQ, ALG, TP, KS * 4 + SH) for ALG 0; (VEC, TQ, ALG, 1, 0) for ALG 1 / 2
template <typename TIn, int VEC, int TQ, bool SMEM>
static void reg_smem(int32_t sketch) {
    registry_add(kernel_key(sketch, VEC, TQ, SMEM ? 1 : 2, 1, 0), &dwconv_launch<TIn, VEC, TQ, SMEM>);
}
template <typename TIn, int VEC, int TQ, int TP, int KS, int SH>
static void reg_win1(int32_t sketch) {
    if constexpr (dw_win_fits(VEC, TQ, TP, KS, SH))  // the same register rule as sketches.cpp
        registry_add(kernel_key(sketch, VEC, TQ, 0, TP, KS * 4 + SH), &dwconv_win_launch<TIn, VEC, TQ, TP, KS, SH>);
}
template <typename TIn, int VEC, int TQ, int TP>
static void reg_win(int32_t sketch) {
    reg_win1<TIn, VEC, TQ, TP, 3, 1>(sketch);
    reg_win1<TIn, VEC, TQ, TP, 3, 2>(sketch);
    reg_win1<TIn, VEC, TQ, TP, 5, 1>(sketch);
    reg_win1<TIn, VEC, TQ, TP, 5, 2>(sketch);
}
template <typename TIn, int VEC, int TQ>
static void reg_tq(int32_t sketch) {
    reg_smem<TIn, VEC, TQ, true>(sketch);
    reg_smem<TIn, VEC, TQ, false>(sketch);
    reg_win<TIn, VEC, TQ, 1>(sketch);
    reg_win<TIn, VEC, TQ, 2>(sketch);
    reg_win<TIn, VEC, TQ, 4>(sketch);
}
template <typename TIn, int VEC>
static void reg_vec(int32_t sketch) {
    reg_tq<TIn, VEC, 1>(sketch);
    reg_tq<TIn, VEC, 2>(sketch);
    reg_tq<TIn, VEC, 4>(sketch);
}

void register_dwconv() {
    reg_vec<float, 1>(SK_SIMT_DWCONV_F32);
    reg_vec<float, 2>(SK_SIMT_DWCONV_F32);
    reg_vec<float, 4>(SK_SIMT_DWCONV_F32);
    reg_vec<__nv_bfloat16, 1>(SK_SIMT_DWCONV_BF16);
    reg_vec<__nv_bfloat16, 2>(SK_SIMT_DWCONV_BF16);
    reg_vec<__nv_bfloat16, 4>(SK_SIMT_DWCONV_BF16);
}

}  // namespace db200
