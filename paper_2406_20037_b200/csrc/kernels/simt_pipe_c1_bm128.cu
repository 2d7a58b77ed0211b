// Explicit instantiations of the cp.async multistage SIMT sketch (generated list, one TU
// per (CONV, BM) so nvcc compiles the family in parallel).
#include "simt_pipe.cuh"

namespace db200 {
void register_simt_pipe_c1_bm128() {
    pipe_register<128, 32, 8, 2, 1, true>();
    pipe_register<128, 32, 8, 4, 1, true>();
    pipe_register<128, 32, 8, 4, 2, true>();
    pipe_register<128, 32, 16, 2, 1, true>();
    pipe_register<128, 32, 16, 4, 1, true>();
    pipe_register<128, 32, 16, 4, 2, true>();
    pipe_register<128, 32, 16, 4, 4, true>();
    pipe_register<128, 32, 32, 2, 1, true>();
    pipe_register<128, 32, 32, 4, 1, true>();
    pipe_register<128, 32, 32, 4, 2, true>();
    pipe_register<128, 32, 32, 4, 4, true>();
    pipe_register<128, 64, 8, 4, 1, true>();
    pipe_register<128, 64, 8, 4, 2, true>();
    pipe_register<128, 64, 16, 4, 1, true>();
    pipe_register<128, 64, 16, 4, 2, true>();
    pipe_register<128, 64, 32, 4, 1, true>();
    pipe_register<128, 64, 32, 4, 2, true>();
    pipe_register<128, 128, 8, 4, 1, true>();
    pipe_register<128, 128, 16, 4, 1, true>();
    pipe_register<128, 128, 32, 4, 1, true>();
}
}  // namespace db200
