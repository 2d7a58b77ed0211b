// registry.cu — (sketch, compile-time knobs) -> launcher table.
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace db200 {

#define DECL_SIMT(c, bm) void register_simt_c##c##_bm##bm();
DECL_SIMT(0, 16) DECL_SIMT(0, 32) DECL_SIMT(0, 64) DECL_SIMT(0, 128)
DECL_SIMT(1, 16) DECL_SIMT(1, 32) DECL_SIMT(1, 64) DECL_SIMT(1, 128)
#define DECL_PIPE(c, bm) void register_simt_pipe_c##c##_bm##bm();
DECL_PIPE(0, 16) DECL_PIPE(0, 32) DECL_PIPE(0, 64) DECL_PIPE(0, 128) DECL_PIPE(1, 16) DECL_PIPE(1, 32) DECL_PIPE(1, 64) DECL_PIPE(1, 128)
void register_tc_gemm();
void register_simt_bf16_conv();
void register_dwconv();
void register_direct_conv();

static std::unordered_map<uint64_t, LaunchFn>& table() {
    static std::unordered_map<uint64_t, LaunchFn> t;
    return t;
}
static std::once_flag g_once;

static void init_all() {
    register_simt_c0_bm16(); register_simt_c0_bm32(); register_simt_c0_bm64(); register_simt_c0_bm128();
    register_simt_c1_bm16(); register_simt_c1_bm32(); register_simt_c1_bm64(); register_simt_c1_bm128();
    register_simt_pipe_c0_bm16(); register_simt_pipe_c0_bm32(); register_simt_pipe_c0_bm64(); register_simt_pipe_c0_bm128();
    register_simt_pipe_c1_bm16(); register_simt_pipe_c1_bm32(); register_simt_pipe_c1_bm64(); register_simt_pipe_c1_bm128();
    register_tc_gemm();
    register_simt_bf16_conv();
    register_dwconv();
    register_direct_conv();
}

uint64_t kernel_key(int32_t sketch, int a, int b, int c, int d, int e) {
    return ((uint64_t)sketch << 50) | ((uint64_t)(a & 1023) << 40) | ((uint64_t)(b & 1023) << 30) |
           ((uint64_t)(c & 1023) << 20) | ((uint64_t)(d & 1023) << 10) | (uint64_t)(e & 1023);
}

void registry_add(uint64_t key, LaunchFn fn) { table()[key] = fn; }

LaunchFn registry_find(uint64_t key) {
    std::call_once(g_once, init_all);
    auto it = table().find(key);
    return it == table().end() ? nullptr : it->second;
}

static std::atomic<int64_t> g_launches{0};
static thread_local bool g_capturing = false;  // launches recorded into a graph are counted at graph launch
void set_capturing(bool on) { g_capturing = on; }
void count_launches(int64_t n) {
    if (!g_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
}
std::atomic<int64_t>* g_launch_counter_ptr() { return &g_launches; }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DB200_NO_PDL");
        return !(e && e[0] && e[0] != '0');
    }();
    return on;
}

}  // namespace db200
