// comm.hpp -- lazily loaded NCCL communicator helpers (see comm.cpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "error.hpp"

namespace rii {
void nccl_unique_id(void *out128);
void *nccl_init(const void *id128, int rank, int world);
void nccl_destroy(void *comm);
void nccl_allgather_u64(void *comm, const uint64_t *send, uint64_t *recv, size_t count, cudaStream_t st);
void nccl_allgather_u8(void *comm, const uint8_t *send, uint8_t *recv, size_t count, cudaStream_t st);
void nccl_allreduce_max_i64(void *comm, const int64_t *send, int64_t *recv, size_t count, cudaStream_t st);
}  // namespace rii
