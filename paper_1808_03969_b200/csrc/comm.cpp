// comm.cpp -- NCCL over NVLink 5 / NVSwitch for the one real exchange step of the
// path (merge of per-GPU top-k lists, and the reconfigure sample).  NCCL is
// loaded lazily with dlopen so the library (and its CPU-side tests) load on
// machines without NCCL or a GPU; world == 1 never touches it.
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace rii {

namespace {
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_api;
std::once_flag g_once;
std::string g_load_error;

void load_api() {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
        g_api.h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
        if (g_api.h) break;
    }
    if (!g_api.h) { g_load_error = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return; }
#define RII_SYM(field, name)                                                         \
    g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(g_api.h, name));     \
    if (!g_api.field) { g_load_error = std::string("missing NCCL symbol ") + name; g_api.h = nullptr; return; }
    RII_SYM(GetUniqueId, "ncclGetUniqueId");
    RII_SYM(CommInitRank, "ncclCommInitRank");
    RII_SYM(CommDestroy, "ncclCommDestroy");
    RII_SYM(AllGather, "ncclAllGather");
    RII_SYM(AllReduce, "ncclAllReduce");
    RII_SYM(GetErrorString, "ncclGetErrorString");
#undef RII_SYM
}

const NcclApi &api() {
    std::call_once(g_once, load_api);
    if (!g_api.h) throw Error(5, g_load_error);
    return g_api;
}

void check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw Error(5, std::string(what) + ": " + api().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(void *out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    check(api().GetUniqueId(&id), "ncclGetUniqueId");
    memcpy(out128, &id, sizeof(id));
}

void *nccl_init(const void *id128, int rank, int world) {
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    check(api().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    return comm;
}

void nccl_destroy(void *comm) {
    if (comm && g_api.h) g_api.CommDestroy(reinterpret_cast<ncclComm_t>(comm));
}

void nccl_allgather_u64(void *comm, const uint64_t *send, uint64_t *recv, size_t count, cudaStream_t st) {
    check(api().AllGather(send, recv, count, ncclUint64, reinterpret_cast<ncclComm_t>(comm), st), "ncclAllGather");
}

void nccl_allgather_u8(void *comm, const uint8_t *send, uint8_t *recv, size_t count, cudaStream_t st) {
    check(api().AllGather(send, recv, count, ncclUint8, reinterpret_cast<ncclComm_t>(comm), st), "ncclAllGather");
}

void nccl_allreduce_max_i64(void *comm, const int64_t *send, int64_t *recv, size_t count, cudaStream_t st) {
    check(api().AllReduce(send, recv, count, ncclInt64, ncclMax, reinterpret_cast<ncclComm_t>(comm), st),
          "ncclAllReduce");
}

}  // namespace rii
