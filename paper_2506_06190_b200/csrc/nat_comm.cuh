// Internal definition of the opaque nat_comm.
#pragma once
#include <nccl.h>

#include "nat_internal.cuh"

struct nat_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, world = 1;
  bool borrowed = false;  // nat_comm_create: the caller owns the ncclComm_t
  // host-staged backend (nat_comm_create_host): the all-gather runs on host memory through
  // the caller's callback; pinned staging owned by the communicator
  nat_allgather_fn host_fn = nullptr;
  void* host_user = nullptr;
  double* staging = nullptr;
  size_t staging_count = 0;
};

namespace nat {
nat_status allgather_inplace(nat_comm* comm, double* buf, size_t count, cudaStream_t s);
// Several in-place all-gathers of `count` doubles per rank (buffers bufs[q], q < nbuf) as
// one NCCL group (one launch for all of them); every rank must pass the same list.
nat_status allgather_inplace_many(nat_comm* comm, double* const* bufs, int nbuf, size_t count, cudaStream_t s);
// matrix-free operator (bem.cu): workspace, per-operator setup, y = (A x) on the op's rows
size_t mf_apply_ws(const nat_bem_mf* op);
nat_status mf_begin(const nat_bem_mf* op, void* ws, size_t ws_bytes, cudaStream_t s);
nat_status mf_apply(const nat_bem_mf* op, void* ws, const double2* x, double2* y, const unsigned long long* skip,
                    cudaStream_t s);
nat_status matvec_internal(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda,
                           const void* x, void* y, cudaStream_t s, const unsigned long long* skip = nullptr);
}  // namespace nat
