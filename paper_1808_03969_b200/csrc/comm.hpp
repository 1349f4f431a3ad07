// comm.hpp -- the one exchange primitive of the multi-GPU path (comm.cpp): an
// all-gather of equal-sized per-rank blocks, over NCCL (device buffers, NVLink /
// NVSwitch) or over a caller-supplied host transport (rii_transport).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/rii.h"
#include "error.hpp"

namespace rii {

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // recv[r * bytes .. (r + 1) * bytes) = rank r's `bytes` bytes at send (device
    // buffers, ordered on st).  Collective: every rank calls it with the same bytes.
    virtual void allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;
    // *recv = max over ranks of *send (count values, device buffers).
    virtual void allreduce_max_i64(const int64_t *send, int64_t *recv, size_t count, cudaStream_t st) = 0;
};

void nccl_unique_id(void *out128);
Comm *nccl_comm_create(const void *id128, int rank, int world);
Comm *host_comm_create(const rii_transport &t, int rank, int world);

}  // namespace rii
