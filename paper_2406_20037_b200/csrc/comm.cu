// comm.cu — the one collective of the hot path: an all-gather of
// fixed-size per-candidate result slots after every measured batch, so that
// every rank holds the identical batch-ordered results and takes the same
// descent step.  NCCL over NVLink/NVSwitch; the communicator is created inside
// the library from a 128-byte unique id the caller broadcasts (e.g. through a
// torch process group).  libnccl is dlopen'ed (the copy torch already loaded,
// RTLD_NOLOAD first) so one NCCL lives in the process.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "internal.hpp"

namespace db200 {

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    const char* env = std::getenv("DROPLET_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        if (!n) continue;
        a.h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);
        if (!a.h) a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (a.h) break;
    }
    if (!a.h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
    a.AllGather = (decltype(a.AllGather))dlsym(a.h, "ncclAllGather");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy;
    return a;
}

tuner_status nccl_fail(ncclResult_t r, const char* what) {
    const char* s = api().GetErrorString ? api().GetErrorString(r) : "?";
    return fail(TUNER_ENCCL, std::string(what) + ": " + s);
}

// One NCCL communicator per (unique id, rank), created on first use and kept for the
// life of the process: every tuner of a process group shares it (a communicator per
// tuner would pay ncclCommInitRank for every layer).
struct NcclShared {
    ncclComm_t comm = nullptr;
    int world = 1;
    char* d_send = nullptr;
    char* d_recv = nullptr;
    int64_t cap = 0;
};

struct NcclComm : Comm {
    NcclShared* sh = nullptr;
    cudaStream_t st = nullptr;
    tuner_status allgather(const void* send, void* recv, int64_t bytes) override {
        if (bytes > sh->cap) {
            if (sh->d_send) cudaFree(sh->d_send);
            if (sh->d_recv) cudaFree(sh->d_recv);
            if (cudaMalloc(&sh->d_send, bytes) != cudaSuccess || cudaMalloc(&sh->d_recv, bytes * sh->world) != cudaSuccess)
                return fail(TUNER_ENOMEM, "NCCL staging buffers");
            sh->cap = bytes;
        }
        if (cudaMemcpyAsync(sh->d_send, send, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
            return fail(TUNER_ECUDA, "H2D of result slots");
        ncclResult_t r = api().AllGather(sh->d_send, sh->d_recv, (size_t)bytes, ncclUint8, sh->comm, st);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
        if (cudaMemcpyAsync(recv, sh->d_recv, bytes * sh->world, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(TUNER_ECUDA, "D2H of gathered slots");
        return TUNER_OK;
    }
};

std::map<std::string, NcclShared*>& comm_cache() {
    static std::map<std::string, NcclShared*> m;
    return m;
}
}  // namespace

tuner_status nccl_unique_id(void* out128) {
    if (!api().ok) return fail(TUNER_ENCCL, "libnccl.so.2 not found (set DROPLET_NCCL_LIB)");
    ncclUniqueId id;
    ncclResult_t r = api().GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, 128);
    return TUNER_OK;
}

tuner_status make_nccl_comm(const void* uid, int rank, int world, void* stream, std::unique_ptr<Comm>& out) {
    if (!api().ok) return fail(TUNER_ENCCL, "libnccl.so.2 not found (set DROPLET_NCCL_LIB)");
    std::string key(static_cast<const char*>(uid), 128);
    key += std::to_string(rank) + "/" + std::to_string(world);
    auto& cache = comm_cache();
    auto it = cache.find(key);
    NcclShared* sh;
    if (it != cache.end()) {
        sh = it->second;
    } else {
        sh = new NcclShared();
        ncclUniqueId id;
        std::memcpy(&id, uid, 128);
        ncclResult_t r = api().CommInitRank(&sh->comm, world, id, rank);
        if (r != ncclSuccess) {
            delete sh;
            return nccl_fail(r, "ncclCommInitRank");
        }
        sh->world = world;
        cache[key] = sh;
    }
    std::unique_ptr<NcclComm> c(new NcclComm());
    c->sh = sh;
    c->st = (cudaStream_t)stream;
    out = std::move(c);
    return TUNER_OK;
}

}  // namespace db200
