// Explicit instantiations of the cp.async multistage SIMT sketch (generated list, one TU
// per (CONV, BM) so nvcc compiles the family in parallel).
#include "simt_pipe.cuh"

namespace db200 {
void register_simt_pipe_c1_bm16() {
    pipe_register<16, 32, 8, 2, 1, true>();
    pipe_register<16, 32, 8, 2, 2, true>();
    pipe_register<16, 32, 8, 4, 1, true>();
    pipe_register<16, 32, 8, 4, 2, true>();
    pipe_register<16, 32, 16, 2, 1, true>();
    pipe_register<16, 32, 16, 2, 2, true>();
    pipe_register<16, 32, 16, 2, 4, true>();
    pipe_register<16, 32, 16, 4, 1, true>();
    pipe_register<16, 32, 16, 4, 2, true>();
    pipe_register<16, 32, 16, 4, 4, true>();
    pipe_register<16, 32, 32, 2, 1, true>();
    pipe_register<16, 32, 32, 2, 2, true>();
    pipe_register<16, 32, 32, 2, 4, true>();
    pipe_register<16, 32, 32, 4, 1, true>();
    pipe_register<16, 32, 32, 4, 2, true>();
    pipe_register<16, 32, 32, 4, 4, true>();
    pipe_register<16, 64, 8, 2, 1, true>();
    pipe_register<16, 64, 8, 2, 2, true>();
    pipe_register<16, 64, 8, 4, 1, true>();
    pipe_register<16, 64, 8, 4, 2, true>();
    pipe_register<16, 64, 16, 2, 1, true>();
    pipe_register<16, 64, 16, 2, 2, true>();
    pipe_register<16, 64, 16, 2, 4, true>();
    pipe_register<16, 64, 16, 4, 1, true>();
    pipe_register<16, 64, 16, 4, 2, true>();
    pipe_register<16, 64, 16, 4, 4, true>();
    pipe_register<16, 64, 32, 2, 1, true>();
    pipe_register<16, 64, 32, 2, 2, true>();
    pipe_register<16, 64, 32, 2, 4, true>();
    pipe_register<16, 64, 32, 4, 1, true>();
    pipe_register<16, 64, 32, 4, 2, true>();
    pipe_register<16, 64, 32, 4, 4, true>();
    pipe_register<16, 128, 8, 2, 1, true>();
    pipe_register<16, 128, 8, 2, 2, true>();
    pipe_register<16, 128, 8, 4, 1, true>();
    pipe_register<16, 128, 8, 4, 2, true>();
    pipe_register<16, 128, 16, 2, 1, true>();
    pipe_register<16, 128, 16, 2, 2, true>();
    pipe_register<16, 128, 16, 4, 1, true>();
    pipe_register<16, 128, 16, 4, 2, true>();
    pipe_register<16, 128, 16, 4, 4, true>();
    pipe_register<16, 128, 32, 2, 1, true>();
    pipe_register<16, 128, 32, 2, 2, true>();
    pipe_register<16, 128, 32, 4, 1, true>();
    pipe_register<16, 128, 32, 4, 2, true>();
    pipe_register<16, 128, 32, 4, 4, true>();
}
}  // namespace db200
