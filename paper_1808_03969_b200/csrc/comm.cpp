// comm.cpp -- the one real exchange step of the multi-GPU path (merge of per-GPU
// top-k lists, the shared u6 bound of a whole-database scan, the reconfigure
// sample): NCCL over NVLink 5 / NVSwitch, or a caller-supplied host transport
// (rii_create_with_transport; e.g. torch.distributed gloo in the multi-process
// tests).  NCCL is loaded lazily with dlopen so the library (and its CPU-side
// tests) load on machines without NCCL or a GPU; world == 1 never touches it.
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

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

namespace {
// NCCL over NVLink 5 / NVSwitch: device buffers, enqueued on the caller's stream.
struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm && g_api.h) g_api.CommDestroy(comm);
    }
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        check(api().AllGather(send, recv, bytes, ncclUint8, comm, st), "ncclAllGather");
    }
    void allreduce_max_i64(const int64_t *send, int64_t *recv, size_t count, cudaStream_t st) override {
        check(api().AllReduce(send, recv, count, ncclInt64, ncclMax, comm, st), "ncclAllReduce");
    }
};

// Caller-supplied host transport (rii_transport): the device block is staged
// through host memory around the callback.  The stream is synchronised first, so
// no kernel of this rank ever waits on another rank's kernels.
struct HostComm final : Comm {
    rii_transport t{};
    void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        std::vector<uint8_t> hs(bytes ? bytes : 1), hr(bytes * (size_t)world + 1);
        if (cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw Error(4, "host transport: device-to-host staging failed");
        if (t.allgather(t.ctx, hs.data(), hr.data(), (uint64_t)bytes) != 0)
            throw Error(5, "host transport: allgather callback failed");
        if (cudaMemcpyAsync(recv, hr.data(), bytes * (size_t)world, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw Error(4, "host transport: host-to-device staging failed");
    }
    void allreduce_max_i64(const int64_t *send, int64_t *recv, size_t count, cudaStream_t st) override {
        std::vector<int64_t> all(count * (size_t)world + 1), h(count + 1);
        int64_t *tmp = nullptr;
        if (cudaMallocAsync(&tmp, count * (size_t)world * 8 + 8, st) != cudaSuccess) throw Error(3, "host transport");
        allgather(send, tmp, count * 8, st);
        cudaMemcpyAsync(all.data(), tmp, count * (size_t)world * 8, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(tmp, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) throw Error(4, "host transport: reduce staging failed");
        for (size_t i = 0; i < count; ++i) {
            h[i] = all[i];
            for (int r = 1; r < world; ++r) h[i] = std::max(h[i], all[(size_t)r * count + i]);
        }
        if (cudaMemcpyAsync(recv, h.data(), count * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            throw Error(4, "host transport: host-to-device staging failed");
    }
};
}  // namespace

Comm *nccl_comm_create(const void *id128, int rank, int world) {
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    auto *c = new NcclComm();
    c->rank = rank;
    c->world = world;
    try {
        check(api().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

Comm *host_comm_create(const rii_transport &t, int rank, int world) {
    if (!t.allgather) throw Error(1, "rii_transport.allgather is NULL");
    auto *c = new HostComm();
    c->t = t;
    c->rank = rank;
    c->world = world;
    return c;
}

}  // namespace rii
