// Internal definition of the opaque nat_comm.
#pragma once
#include <nccl.h>

#include "nat_internal.cuh"

struct nat_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, world = 1;
};

namespace nat {
nat_status allgather_inplace(nat_comm* comm, double* buf, size_t count, cudaStream_t s);
nat_status matvec_internal(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda,
                           const void* x, void* y, cudaStream_t s, const unsigned long long* skip = nullptr);
}  // namespace nat
