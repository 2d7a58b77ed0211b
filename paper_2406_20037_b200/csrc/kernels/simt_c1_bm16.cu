// Explicit instantiations of the SIMT fp32 sketch (generated list, one TU per (CONV, BM)
// so nvcc compiles the family in parallel).
#include "simt_gemm.cuh"

namespace db200 {
void register_simt_c1_bm16() {
    simt_register<16, 16, 4, 2, 1, true>(); simt_register<16, 16, 4, 2, 2, true>(); simt_register<16, 16, 4, 2, 4, true>(); simt_register<16, 16, 4, 2, 8, true>();
    simt_register<16, 16, 4, 4, 1, true>(); simt_register<16, 16, 4, 4, 2, true>(); simt_register<16, 16, 4, 4, 4, true>(); simt_register<16, 16, 4, 4, 8, true>();
    simt_register<16, 16, 4, 8, 1, true>(); simt_register<16, 16, 4, 8, 2, true>(); simt_register<16, 16, 4, 8, 4, true>(); simt_register<16, 16, 4, 8, 8, true>();
    simt_register<16, 16, 8, 2, 1, true>(); simt_register<16, 16, 8, 2, 2, true>(); simt_register<16, 16, 8, 2, 4, true>(); simt_register<16, 16, 8, 2, 8, true>();
    simt_register<16, 16, 8, 4, 1, true>(); simt_register<16, 16, 8, 4, 2, true>(); simt_register<16, 16, 8, 4, 4, true>(); simt_register<16, 16, 8, 4, 8, true>();
    simt_register<16, 16, 8, 8, 1, true>(); simt_register<16, 16, 8, 8, 2, true>(); simt_register<16, 16, 8, 8, 4, true>(); simt_register<16, 16, 8, 8, 8, true>();
    simt_register<16, 16, 16, 2, 1, true>(); simt_register<16, 16, 16, 2, 2, true>(); simt_register<16, 16, 16, 2, 4, true>(); simt_register<16, 16, 16, 2, 8, true>();
    simt_register<16, 16, 16, 4, 1, true>(); simt_register<16, 16, 16, 4, 2, true>(); simt_register<16, 16, 16, 4, 4, true>(); simt_register<16, 16, 16, 4, 8, true>();
    simt_register<16, 16, 16, 8, 1, true>(); simt_register<16, 16, 16, 8, 2, true>(); simt_register<16, 16, 16, 8, 4, true>(); simt_register<16, 16, 16, 8, 8, true>();
    simt_register<16, 16, 32, 2, 1, true>(); simt_register<16, 16, 32, 2, 2, true>(); simt_register<16, 16, 32, 2, 4, true>(); simt_register<16, 16, 32, 2, 8, true>();
    simt_register<16, 16, 32, 4, 1, true>(); simt_register<16, 16, 32, 4, 2, true>(); simt_register<16, 16, 32, 4, 4, true>(); simt_register<16, 16, 32, 4, 8, true>();
    simt_register<16, 16, 32, 8, 1, true>(); simt_register<16, 16, 32, 8, 2, true>(); simt_register<16, 16, 32, 8, 4, true>(); simt_register<16, 16, 32, 8, 8, true>();
    simt_register<16, 32, 4, 2, 1, true>(); simt_register<16, 32, 4, 2, 2, true>(); simt_register<16, 32, 4, 2, 4, true>(); simt_register<16, 32, 4, 2, 8, true>();
    simt_register<16, 32, 4, 4, 1, true>(); simt_register<16, 32, 4, 4, 2, true>(); simt_register<16, 32, 4, 4, 4, true>(); simt_register<16, 32, 4, 4, 8, true>();
    simt_register<16, 32, 4, 8, 1, true>(); simt_register<16, 32, 4, 8, 2, true>(); simt_register<16, 32, 4, 8, 4, true>(); simt_register<16, 32, 4, 8, 8, true>();
    simt_register<16, 32, 8, 2, 1, true>(); simt_register<16, 32, 8, 2, 2, true>(); simt_register<16, 32, 8, 2, 4, true>(); simt_register<16, 32, 8, 2, 8, true>();
    simt_register<16, 32, 8, 4, 1, true>(); simt_register<16, 32, 8, 4, 2, true>(); simt_register<16, 32, 8, 4, 4, true>(); simt_register<16, 32, 8, 4, 8, true>();
    simt_register<16, 32, 8, 8, 1, true>(); simt_register<16, 32, 8, 8, 2, true>(); simt_register<16, 32, 8, 8, 4, true>(); simt_register<16, 32, 8, 8, 8, true>();
    simt_register<16, 32, 16, 2, 1, true>(); simt_register<16, 32, 16, 2, 2, true>(); simt_register<16, 32, 16, 2, 4, true>(); simt_register<16, 32, 16, 2, 8, true>();
    simt_register<16, 32, 16, 4, 1, true>(); simt_register<16, 32, 16, 4, 2, true>(); simt_register<16, 32, 16, 4, 4, true>(); simt_register<16, 32, 16, 4, 8, true>();
    simt_register<16, 32, 16, 8, 1, true>(); simt_register<16, 32, 16, 8, 2, true>(); simt_register<16, 32, 16, 8, 4, true>(); simt_register<16, 32, 16, 8, 8, true>();
    simt_register<16, 32, 32, 2, 1, true>(); simt_register<16, 32, 32, 2, 2, true>(); simt_register<16, 32, 32, 2, 4, true>(); simt_register<16, 32, 32, 2, 8, true>();
    simt_register<16, 32, 32, 4, 1, true>(); simt_register<16, 32, 32, 4, 2, true>(); simt_register<16, 32, 32, 4, 4, true>(); simt_register<16, 32, 32, 4, 8, true>();
    simt_register<16, 32, 32, 8, 1, true>(); simt_register<16, 32, 32, 8, 2, true>(); simt_register<16, 32, 32, 8, 4, true>(); simt_register<16, 32, 32, 8, 8, true>();
    simt_register<16, 64, 4, 2, 1, true>(); simt_register<16, 64, 4, 2, 2, true>(); simt_register<16, 64, 4, 2, 4, true>(); simt_register<16, 64, 4, 2, 8, true>();
    simt_register<16, 64, 4, 4, 1, true>(); simt_register<16, 64, 4, 4, 2, true>(); simt_register<16, 64, 4, 4, 4, true>(); simt_register<16, 64, 4, 4, 8, true>();
    simt_register<16, 64, 4, 8, 1, true>(); simt_register<16, 64, 4, 8, 2, true>(); simt_register<16, 64, 4, 8, 4, true>(); simt_register<16, 64, 4, 8, 8, true>();
    simt_register<16, 64, 8, 2, 1, true>(); simt_register<16, 64, 8, 2, 2, true>(); simt_register<16, 64, 8, 2, 4, true>(); simt_register<16, 64, 8, 2, 8, true>();
    simt_register<16, 64, 8, 4, 1, true>(); simt_register<16, 64, 8, 4, 2, true>(); simt_register<16, 64, 8, 4, 4, true>(); simt_register<16, 64, 8, 4, 8, true>();
    simt_register<16, 64, 8, 8, 1, true>(); simt_register<16, 64, 8, 8, 2, true>(); simt_register<16, 64, 8, 8, 4, true>(); simt_register<16, 64, 8, 8, 8, true>();
    simt_register<16, 64, 16, 2, 1, true>(); simt_register<16, 64, 16, 2, 2, true>(); simt_register<16, 64, 16, 2, 4, true>(); simt_register<16, 64, 16, 2, 8, true>();
    simt_register<16, 64, 16, 4, 1, true>(); simt_register<16, 64, 16, 4, 2, true>(); simt_register<16, 64, 16, 4, 4, true>(); simt_register<16, 64, 16, 4, 8, true>();
    simt_register<16, 64, 16, 8, 1, true>(); simt_register<16, 64, 16, 8, 2, true>(); simt_register<16, 64, 16, 8, 4, true>(); simt_register<16, 64, 16, 8, 8, true>();
    simt_register<16, 64, 32, 2, 1, true>(); simt_register<16, 64, 32, 2, 2, true>(); simt_register<16, 64, 32, 2, 4, true>(); simt_register<16, 64, 32, 2, 8, true>();
    simt_register<16, 64, 32, 4, 1, true>(); simt_register<16, 64, 32, 4, 2, true>(); simt_register<16, 64, 32, 4, 4, true>(); simt_register<16, 64, 32, 4, 8, true>();
    simt_register<16, 64, 32, 8, 1, true>(); simt_register<16, 64, 32, 8, 2, true>(); simt_register<16, 64, 32, 8, 4, true>(); simt_register<16, 64, 32, 8, 8, true>();
    simt_register<16, 128, 4, 2, 1, true>(); simt_register<16, 128, 4, 2, 2, true>(); simt_register<16, 128, 4, 2, 4, true>(); simt_register<16, 128, 4, 2, 8, true>();
    simt_register<16, 128, 4, 4, 1, true>(); simt_register<16, 128, 4, 4, 2, true>(); simt_register<16, 128, 4, 4, 4, true>(); simt_register<16, 128, 4, 4, 8, true>();
    simt_register<16, 128, 4, 8, 1, true>(); simt_register<16, 128, 4, 8, 2, true>(); simt_register<16, 128, 4, 8, 4, true>(); simt_register<16, 128, 4, 8, 8, true>();
    simt_register<16, 128, 8, 2, 1, true>(); simt_register<16, 128, 8, 2, 2, true>(); simt_register<16, 128, 8, 2, 4, true>(); simt_register<16, 128, 8, 2, 8, true>();
    simt_register<16, 128, 8, 4, 1, true>(); simt_register<16, 128, 8, 4, 2, true>(); simt_register<16, 128, 8, 4, 4, true>(); simt_register<16, 128, 8, 4, 8, true>();
    simt_register<16, 128, 8, 8, 1, true>(); simt_register<16, 128, 8, 8, 2, true>(); simt_register<16, 128, 8, 8, 4, true>(); simt_register<16, 128, 8, 8, 8, true>();
    simt_register<16, 128, 16, 2, 1, true>(); simt_register<16, 128, 16, 2, 2, true>(); simt_register<16, 128, 16, 2, 4, true>(); simt_register<16, 128, 16, 2, 8, true>();
    simt_register<16, 128, 16, 4, 1, true>(); simt_register<16, 128, 16, 4, 2, true>(); simt_register<16, 128, 16, 4, 4, true>(); simt_register<16, 128, 16, 4, 8, true>();
    simt_register<16, 128, 16, 8, 1, true>(); simt_register<16, 128, 16, 8, 2, true>(); simt_register<16, 128, 16, 8, 4, true>(); simt_register<16, 128, 16, 8, 8, true>();
    simt_register<16, 128, 32, 2, 1, true>(); simt_register<16, 128, 32, 2, 2, true>(); simt_register<16, 128, 32, 2, 4, true>(); simt_register<16, 128, 32, 2, 8, true>();
    simt_register<16, 128, 32, 4, 1, true>(); simt_register<16, 128, 32, 4, 2, true>(); simt_register<16, 128, 32, 4, 4, true>(); simt_register<16, 128, 32, 4, 8, true>();
    simt_register<16, 128, 32, 8, 1, true>(); simt_register<16, 128, 32, 8, 2, true>(); simt_register<16, 128, 32, 8, 4, true>(); simt_register<16, 128, 32, 8, 8, true>();
}
}  // namespace db200
