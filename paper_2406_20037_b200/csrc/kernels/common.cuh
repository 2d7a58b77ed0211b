// common.cuh — launch context and registry shared by the kernel family.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../shape.hpp"

namespace db200 {

// Everything a candidate launch needs; built by the harness per launch.
struct LaunchCtx {
    const ShapeInfo* sh;
    const void* x;
    const void* w;
    void* y;
    int split;             // runtime SPLIT_K knob
    int vec;               // runtime VEC knob (SIMT)
    int stages;            // runtime STAGES knob (SIMT)
    int sched;             // runtime SCHED knob (tcgen05: 0 tiles, 1 stream-K)
    cudaStream_t stream;
    int num_sms;
    int dims[3] = {1, 1, 1};  // runtime thread-block shape knobs (depthwise: CT, QT, PT)
    int raster = 0;           // runtime tile order (tcgen05): 0 = M fastest, 1 = N fastest
    const StreamKScratch* sk = nullptr;  // stream-K workspace of the launching handle (SCHED >= 1)
    int occ = 0;                         // runtime OCC knob (SIMT pipe): 0 = a CTA per unit, k = k CTAs/SM persistent
    int red = 0;                         // runtime RED knob (SIMT pipe): split-K by 0 = atomics, 1 = cluster DSMEM
    int epi = 1;                         // runtime EPI knob (tcgen05): epilogue staging buffer sets per warp
};

typedef cudaError_t (*LaunchFn)(const LaunchCtx&);

// Registry of compiled instantiations: key = (sketch, compile-time knob values).
uint64_t kernel_key(int32_t sketch, int a, int b, int c, int d, int e);
void registry_add(uint64_t key, LaunchFn fn);
LaunchFn registry_find(uint64_t key);

// Counter of candidate-kernel launches (graph nodes included).
void count_launches(int64_t n);
void set_capturing(bool on);

// Dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize) once per
// (kernel instantiation, device): the attribute is per device, so a process driving several
// devices sets it on each (one bit per device ordinal < 64 in the instantiation's mask).
template <typename K>
inline cudaError_t smem_optin(std::atomic<unsigned long long>& mask, K kern, int bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Split-K zeroing as a kernel that lets the partial-sum kernel launch early (programmatic
// dependent launch): the dependent kernel stages and multiplies while Y is being zeroed and
// waits (griddep_wait) only before its first atomic.  Replaces cudaMemsetAsync + full
// stream serialisation: the zeroing node's launch and run time leave the critical path.
cudaError_t zero_for_splitk(float* y, long long n, cudaStream_t st);
// launch attribute for the dependent kernel (cudaLaunchKernelEx); DB200_NO_PDL=1 turns the
// early launch off (plain stream serialisation) for A/B timing
bool pdl_enabled();
inline void pdl_attr(cudaLaunchAttribute& a) {
    a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a.val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
}
// wait until the prerequisite grid (the zeroing kernel) has completed and its writes are
// visible; returns at once for a kernel launched without a programmatic dependency
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace db200
