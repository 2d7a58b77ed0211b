// umma_shift_probe.cu — does a tcgen05.mma A operand (K-major, SWIZZLE_128B) whose start
// address is shifted by s whole 128-byte rows (not 1024-B aligned) read rows s..s+127?
// The halo-tile conv sketch feeds filter tap (r, s) as such a shifted view of one staged
// input window.  Tests both readings of the descriptor's 3-bit "matrix base offset"
// (bits 49-51): left 0, or set to (start >> 7) & 7.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_20037_b200/csrc/kernels \
//        tools/umma_shift_probe.cu -o build/umma_shift_probe -lcuda && build/umma_shift_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace db200;

constexpr int ROWS = 160, M = 128, N = 64, K = 64;

__device__ __forceinline__ uint64_t desc_shifted(uint32_t saddr, int mode) {
    uint64_t d = tc::sdesc_sw128(saddr);
    if (mode == 1) d |= (uint64_t)((saddr >> 7) & 7) << 49;
    return d;
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int shift, int mode) {
    extern __shared__ uint8_t raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = base;                 // ROWS x 128 B
    uint8_t* sb = base + ROWS * 128;    // N x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // 128B swizzle (absolute smem address bits [4:6] ^= [7:9]), base 1024-aligned
    for (int e = tid; e < ROWS * 8; e += blockDim.x) {
        const int row = e / 8, ch = e % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(A + row * 64 + ch * 8);
        *reinterpret_cast<uint4*>(sa + row * 128 + ((ch ^ (row & 7)) * 16)) = v;
    }
    for (int e = tid; e < N * 8; e += blockDim.x) {
        const int row = e / 8, ch = e % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(B + row * 64 + ch * 8);
        *reinterpret_cast<uint4*>(sb + row * 128 + ((ch ^ (row & 7)) * 16)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        tc::mbar_init(tc::smem_u32(&bar), 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<64>(tc::smem_u32(&tslot));
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16(M, N);
        for (int k = 0; k < K / 16; ++k) {
            const uint32_t a_addr = tc::smem_u32(sa) + shift * 128 + k * 32;
            const uint32_t b_addr = tc::smem_u32(sb) + k * 32;
            tc::umma_bf16(tmem, desc_shifted(a_addr, mode), tc::sdesc_sw128(b_addr), idesc, k > 0 ? 1u : 0u);
        }
        tc::umma_commit(tc::smem_u32(&bar));
    }
    tc::mbar_wait(tc::smem_u32(&bar), 0);
    tc::tc_fence_after();
    for (int c = 0; c < N; c += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
        tc::tmem_ld_wait();
        for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<64>(tmem);
}

int main() {
    std::vector<__nv_bfloat16> hA(ROWS * 64), hB(N * 64);
    std::vector<float> fA(ROWS * 64), fB(N * 64);
    for (int i = 0; i < ROWS; ++i)
        for (int k = 0; k < 64; ++k) {
            fA[i * 64 + k] = (float)((i * 7 + k * 3) % 13 - 6);
            hA[i * 64 + k] = __float2bfloat16(fA[i * 64 + k]);
        }
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < 64; ++k) {
            fB[n * 64 + k] = (float)((n * 5 + k * 11) % 9 - 4);
            hB[n * 64 + k] = __float2bfloat16(fB[n * 64 + k]);
        }
    __nv_bfloat16 *dA, *dB;
    float* dD;
    cudaMalloc(&dA, hA.size() * 2);
    cudaMalloc(&dB, hB.size() * 2);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    const int smem = 1024 + (ROWS + N) * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> hD(M * N);
    int shifts[] = {0, 1, 2, 3, 7, 8, 9, 17, 31};
    for (int mode = 0; mode < 2; ++mode)
        for (int s : shifts) {
            cudaMemset(dD, 0, M * N * 4);
            probe<<<1, 128, smem>>>(dA, dB, dD, s, mode);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d shift %2d: CUDA error %s\n", mode, s, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            int bad = 0, best_match = -1;
            for (int i = 0; i < M; ++i)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) ref += (double)fA[(i + s) * 64 + k] * fB[n * 64 + k];
                    const double err = std::abs(ref - hD[i * N + n]);
                    if (err > maxerr) maxerr = err;
                    bad += err > 0;
                }
            // which shift does the result actually match (row 0 of D against every candidate row)?
            for (int t = 0; t + M <= ROWS && best_match < 0; ++t) {
                bool ok = true;
                for (int i = 0; i < M && ok; ++i)
                    for (int n = 0; n < N && ok; ++n) {
                        double ref = 0;
                        for (int k = 0; k < K; ++k) ref += (double)fA[(i + t) * 64 + k] * fB[n * 64 + k];
                        ok = ref == hD[i * N + n];
                    }
                if (ok) best_match = t;
            }
            printf("mode %d (base offset %s) shift %2d: max abs err %.1f, %d/%d wrong, result == rows %d..\n", mode,
                   mode ? "(start>>7)&7" : "0", s, maxerr, bad, M * N, best_match);
        }
    return 0;
}
