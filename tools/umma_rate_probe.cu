// umma_rate_probe.cu — cycles per tcgen05.mma (kind::f16, cta_group::1, M = 128, K = 16) issued
// back to back by one thread, for N = 64 / 128 / 256, with (a) descriptors advanced by a constant
// (the cheapest issue loop) and (b) descriptors built per MMA from a runtime ring index
// (it % stages, it / stages: the integer divisions of a runtime-STAGES issue loop).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_20037_b200/csrc/kernels \
//        tools/umma_rate_probe.cu -o ab/umma_rate_probe -lcuda && ab/umma_rate_probe
#include <cstdio>

#include "tc_common.cuh"

using namespace db200;

template <int N, int MODE>
__global__ void probe(int iters, int stages, unsigned long long* out, int fill) {
    extern __shared__ uint8_t raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    // operands: zeros, or (FILL = 1) pseudo-random bf16 in [-1, 1) -- the tensor pipe's rate may
    // depend on the data it switches
    for (int i = tid; i < (8 * 16384) / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u;
        h ^= h >> 15;
        h *= 2246822519u;
        const uint32_t lo = 0x3F80u | (h & 0x807Fu), hi = 0x3F00u | ((h >> 16) & 0x807Fu);
        reinterpret_cast<uint32_t*>(base)[i] = fill ? (lo | (hi << 16)) : 0u;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        tc::mbar_init(tc::smem_u32(&bar), 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<256>(tc::smem_u32(&tslot));
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tslot;
    if (tid == 0) {
        constexpr uint32_t idesc = tc::idesc_bf16(128, N);
        const uint32_t sa = tc::smem_u32(base), sb = sa + 16384;
        unsigned long long t0 = clock64();
        if (MODE == 0) {
            uint64_t da = tc::sdesc_sw128(sa), db = tc::sdesc_sw128(sb);
            for (int i = 0; i < iters; ++i) {
                tc::umma_bf16(tmem, da + ((i & 3) << 1), db + ((i & 3) << 1), idesc, 1u);
            }
        } else {
            for (int it = 0; it < iters; ++it) {
                const int s = (it / 4) % stages;
                const uint32_t ph = (uint32_t)((it / 4) / stages) & 1u;
                const uint32_t a = sa + (uint32_t)(s * 1024) + (it & 3) * 32 + ph * 0;
                tc::umma_bf16(tmem, tc::sdesc_sw128(a), tc::sdesc_sw128(sb + (it & 3) * 32), idesc, 1u);
            }
        }
        unsigned long long t1 = clock64();
        tc::umma_commit(tc::smem_u32(&bar));
        tc::mbar_wait(tc::smem_u32(&bar), 0);
        unsigned long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

template <int N, int MODE>
void run(int iters, unsigned long long* d, int fill) {
    const int smem = 1024 + 8 * 16384;
    cudaFuncSetAttribute(probe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long h[2];
    for (int rep = 0; rep < 2; ++rep) {
        probe<N, MODE><<<1, 128, smem>>>(iters, 4, d, fill);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d mode %d (%s), %s operands: issue %.1f cyc/MMA, complete %.1f cyc/MMA (floor 128*N/256 = %d)\n", N,
           MODE, MODE ? "ring index with runtime divisions" : "constant descriptor step", fill ? "random" : "zero",
           (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const int iters = 4096;
    for (int fill = 0; fill < 2; ++fill) {
        run<64, 0>(iters, d, fill);
        run<64, 1>(iters, d, fill);
        run<128, 0>(iters, d, fill);
        run<256, 0>(iters, d, fill);
    }
    return 0;
}
