// tc_gemm.cu — sketch TC_GEMM_BF16 (tcgen05 / TMEM / TMA).  Filled in below.
#include "common.cuh"

namespace db200 {
void register_tc_gemm() {}
}  // namespace db200
