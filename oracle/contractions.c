/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU direct loops for the contractions the
 * tuner's kernel family computes.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant with paper_2406_20037_b200/.
 *
 * Source of the definition: PAPER.md Def. 2.1 (lines 105-114): "The naive
 * implementation of a kernel replaces each linear index in the abstract
 * representation of the kernel with a loop."  Each function below is exactly
 * that naive loop nest, accumulated in fp64, one output at a time, with no
 * blocking, fusion or reordering.  The loop over outputs is split across
 * OpenMP threads only (each output's sum keeps its plain k / (r,s,c) order).
 *
 * Operation semantics (DESIGN.md "readings" R-C1..R-C3):
 *   dense : Y[m,n]     = sum_k X[m,k] * W[n,k]                (W is [N,K])
 *   bmm   : Y[b,m,n]   = sum_k X[b,m,k] * W[b,n,k]
 *   conv2d: Y[n,p,q,k] = sum_{r<R,s<S,c<C} X[n, p*sh-ph+r*dh, q*sw-pw+s*dw, c]
 *                                          * W[k,r,s,c]      (NHWC / KRSC / NPQK,
 *           out-of-bounds taps contribute 0; P = (H+2ph-dh(R-1)-1)/sh + 1, Q alike)
 *   grouped conv2d (G groups; depthwise = G = C = K, the MobileNet/MnasNet/ShuffleNet/
 *           EfficientNet layers of SURVEY §8(f) f4):
 *           Y[n,p,q,k] = sum_{r<R,s<S,c<C/G} X[n, p*sh-ph+r*dh, q*sw-pw+s*dw, g*(C/G)+c]
 *                                          * W[k,r,s,c],  g = k / (K/G)   (W is [K][R][S][C/G])
 * Every function also produces A = the same loops over |X|*|W| (the forward
 * error denominator used by the verification metric, DESIGN.md R-V1).
 */
#include <math.h>
#include <stdint.h>

/* dense / batch_matmul: Y[b,m,n] = sum_k X[b,m,k] W[b,n,k]  (b = 1 for dense) */
void oracle_bmm_f64(const double* X, const double* W, double* Y, double* A,
                    int64_t B, int64_t M, int64_t N, int64_t K) {
    int64_t total = B * M * N;
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < total; ++o) {
        int64_t b = o / (M * N);
        int64_t m = (o / N) % M;
        int64_t n = o % N;
        const double* x = X + (b * M + m) * K;
        const double* w = W + (b * N + n) * K;
        double acc = 0.0, aab = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            acc += x[k] * w[k];
            aab += fabs(x[k]) * fabs(w[k]);
        }
        Y[o] = acc;
        if (A) A[o] = aab;
    }
}

static int64_t out_extent(int64_t in, int64_t pad, int64_t dil, int64_t ker, int64_t stride) {
    return (in + 2 * pad - dil * (ker - 1) - 1) / stride + 1;
}

/* one conv2d output, plain (r, s, c) loop order */
static void conv_one(const double* X, const double* W, double* y, double* a,
                     int64_t H, int64_t Wd, int64_t C, int64_t R, int64_t S,
                     int64_t sh, int64_t sw, int64_t ph, int64_t pw, int64_t dh, int64_t dw,
                     int64_t n, int64_t p, int64_t q, int64_t k) {
    double acc = 0.0, aab = 0.0;
    for (int64_t r = 0; r < R; ++r) {
        int64_t h = p * sh - ph + r * dh;
        for (int64_t s = 0; s < S; ++s) {
            int64_t w = q * sw - pw + s * dw;
            if (h < 0 || h >= H || w < 0 || w >= Wd) continue; /* zero padding */
            const double* xp = X + ((n * H + h) * Wd + w) * C;
            const double* wp = W + ((k * R + r) * S + s) * C;
            for (int64_t c = 0; c < C; ++c) {
                acc += xp[c] * wp[c];
                aab += fabs(xp[c]) * fabs(wp[c]);
            }
        }
    }
    *y = acc;
    if (a) *a = aab;
}

/* conv2d, groups = 1, NHWC input, KRSC weight, NPQK output */
void oracle_conv2d_f64(const double* X, const double* W, double* Y, double* A,
                       int64_t N, int64_t H, int64_t Wd, int64_t C, int64_t K,
                       int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                       int64_t pw, int64_t dh, int64_t dw) {
    int64_t P = out_extent(H, ph, dh, R, sh);
    int64_t Q = out_extent(Wd, pw, dw, S, sw);
    int64_t total = N * P * Q * K;
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < total; ++o) {
        int64_t k = o % K;
        int64_t q = (o / K) % Q;
        int64_t p = (o / (K * Q)) % P;
        int64_t n = o / (K * Q * P);
        conv_one(X, W, Y + o, A ? A + o : 0, H, Wd, C, R, S, sh, sw, ph, pw, dh, dw, n, p, q, k);
    }
}

/* selected conv2d outputs only (for full-size sampled parity): idx[i] = linear NPQK index */
void oracle_conv2d_at_f64(const double* X, const double* W, const int64_t* idx, int64_t cnt,
                          double* Y, double* A, int64_t N, int64_t H, int64_t Wd, int64_t C,
                          int64_t K, int64_t R, int64_t S, int64_t sh, int64_t sw, int64_t ph,
                          int64_t pw, int64_t dh, int64_t dw) {
    int64_t P = out_extent(H, ph, dh, R, sh);
    int64_t Q = out_extent(Wd, pw, dw, S, sw);
    (void)N;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        int64_t o = idx[i];
        int64_t k = o % K;
        int64_t q = (o / K) % Q;
        int64_t p = (o / (K * Q)) % P;
        int64_t n = o / (K * Q * P);
        conv_one(X, W, Y + i, A ? A + i : 0, H, Wd, C, R, S, sh, sw, ph, pw, dh, dw, n, p, q, k);
    }
}

/* one grouped-conv2d output: the plain (r, s, c) loop over the group's C/G channels */
static void gconv_one(const double* X, const double* W, double* y, double* a,
                      int64_t H, int64_t Wd, int64_t C, int64_t K, int64_t G, int64_t R, int64_t S,
                      int64_t sh, int64_t sw, int64_t ph, int64_t pw, int64_t dh, int64_t dw,
                      int64_t n, int64_t p, int64_t q, int64_t k) {
    int64_t cg = C / G;          /* input channels per group */
    int64_t g = k / (K / G);     /* the group output channel k belongs to */
    double acc = 0.0, aab = 0.0;
    for (int64_t r = 0; r < R; ++r) {
        int64_t h = p * sh - ph + r * dh;
        for (int64_t s = 0; s < S; ++s) {
            int64_t w = q * sw - pw + s * dw;
            if (h < 0 || h >= H || w < 0 || w >= Wd) continue; /* zero padding */
            const double* xp = X + ((n * H + h) * Wd + w) * C + g * cg;
            const double* wp = W + ((k * R + r) * S + s) * cg;
            for (int64_t c = 0; c < cg; ++c) {
                acc += xp[c] * wp[c];
                aab += fabs(xp[c]) * fabs(wp[c]);
            }
        }
    }
    *y = acc;
    if (a) *a = aab;
}

/* grouped conv2d (G | C, G | K), NHWC input, W [K][R][S][C/G], NPQK output; with
   idx != NULL only the outputs at the linear NPQK indices idx[0..cnt) */
void oracle_gconv2d_f64(const double* X, const double* W, const int64_t* idx, int64_t cnt,
                        double* Y, double* A, int64_t N, int64_t H, int64_t Wd, int64_t C,
                        int64_t K, int64_t G, int64_t R, int64_t S, int64_t sh, int64_t sw,
                        int64_t ph, int64_t pw, int64_t dh, int64_t dw) {
    int64_t P = out_extent(H, ph, dh, R, sh);
    int64_t Q = out_extent(Wd, pw, dw, S, sw);
    int64_t total = idx ? cnt : N * P * Q * K;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; ++i) {
        int64_t o = idx ? idx[i] : i;
        int64_t k = o % K;
        int64_t q = (o / K) % Q;
        int64_t p = (o / (K * Q)) % P;
        int64_t n = o / (K * Q * P);
        gconv_one(X, W, Y + i, A ? A + i : 0, H, Wd, C, K, G, R, S, sh, sw, ph, pw, dh, dw, n, p, q, k);
    }
}

/* selected bmm outputs only: idx[i] = linear (b, m, n) index */
void oracle_bmm_at_f64(const double* X, const double* W, const int64_t* idx, int64_t cnt,
                       double* Y, double* A, int64_t B, int64_t M, int64_t N, int64_t K) {
    (void)B;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; ++i) {
        int64_t o = idx[i];
        int64_t b = o / (M * N);
        int64_t m = (o / N) % M;
        int64_t n = o % N;
        const double* x = X + (b * M + m) * K;
        const double* w = W + (b * N + n) * K;
        double acc = 0.0, aab = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            acc += x[k] * w[k];
            aab += fabs(x[k]) * fabs(w[k]);
        }
        Y[i] = acc;
        if (A) A[i] = aab;
    }
}

int oracle_num_threads(void) {
    int n = 1;
#pragma omp parallel
    {
#pragma omp single
        {
#ifdef _OPENMP
            extern int omp_get_num_threads(void);
            n = omp_get_num_threads();
#endif
        }
    }
    return n;
}
