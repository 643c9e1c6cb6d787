// NCCL communicator for the row-sharded GMRES (NVLink 5 / NVSwitch inside one box).
// Rank 0 creates the ncclUniqueId; the caller broadcasts its 128 bytes with
// torch.distributed and every rank builds its own communicator from it.
#include <nccl.h>

#include <cstring>

#include "nat_comm.cuh"
#include "nat_internal.cuh"

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");

extern "C" nat_status nat_comm_unique_id(uint8_t* id) {
  NAT_TRACE();
  NAT_REQUIRE(id, "id must be a host buffer of 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nat::fail(NAT_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(id, &u, sizeof u);
  return NAT_OK;
}

extern "C" nat_status nat_comm_create_from_id(nat_comm** comm, const uint8_t* id, int rank, int world) {
  NAT_TRACE();
  NAT_REQUIRE(comm && id, "comm and id must be non-null");
  NAT_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank %d / world %d", rank, world);
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  nat_comm* c = new nat_comm();
  c->rank = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nat::fail(NAT_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *comm = c;
  return NAT_OK;
}

// Wraps a caller-owned ncclComm_t (e.g. the one torch.distributed's NCCL backend holds);
// nat_comm_destroy never destroys a borrowed communicator.  NULL => world 1.
extern "C" nat_status nat_comm_create(nat_comm** comm, void* nccl_comm, int rank, int world) {
  NAT_TRACE();
  NAT_REQUIRE(comm, "comm must be non-null");
  NAT_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank %d / world %d", rank, world);
  NAT_REQUIRE(nccl_comm || world == 1, "a NULL ncclComm_t needs world == 1");
  if (nccl_comm) {
    int n = 0, rk = 0;
    ncclResult_t r = ncclCommCount((ncclComm_t)nccl_comm, &n);
    if (r == ncclSuccess) r = ncclCommUserRank((ncclComm_t)nccl_comm, &rk);
    if (r != ncclSuccess) return nat::fail(NAT_ERR_NCCL, "ncclCommCount/UserRank: %s", ncclGetErrorString(r));
    NAT_REQUIRE(n == world && rk == rank, "ncclComm_t has rank %d of %d, expected %d of %d", rk, n, rank, world);
  }
  nat_comm* c = new nat_comm();
  c->nccl = (ncclComm_t)nccl_comm;
  c->rank = rank;
  c->world = world;
  c->borrowed = true;
  *comm = c;
  return NAT_OK;
}

// Host-staged communicator (no NCCL): every all-gather copies the rank's block to pinned
// host memory, calls fn (which must leave all `world` blocks in the buffer, e.g. through
// torch.distributed on a gloo group), and copies the full buffer back.  Kernels never wait
// on each other across ranks, so ranks may share one GPU (tests of the world > 1 path).
extern "C" nat_status nat_comm_create_host(nat_comm** comm, int rank, int world, nat_allgather_fn fn, void* user) {
  NAT_TRACE();
  NAT_REQUIRE(comm && fn, "comm and fn must be non-null");
  NAT_REQUIRE(world >= 1 && rank >= 0 && rank < world, "bad rank %d / world %d", rank, world);
  nat_comm* c = new nat_comm();
  c->rank = rank;
  c->world = world;
  c->host_fn = fn;
  c->host_user = user;
  *comm = c;
  return NAT_OK;
}

extern "C" nat_status nat_comm_destroy(nat_comm* comm) {
  NAT_TRACE();
  if (!comm) return NAT_OK;
  if (comm->staging) cudaFreeHost(comm->staging);
  ncclResult_t r = (comm->borrowed || !comm->nccl) ? ncclSuccess : ncclCommDestroy(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return nat::fail(NAT_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return NAT_OK;
}

namespace nat {
namespace {
nat_status host_allgather(nat_comm* comm, double* buf, size_t count, cudaStream_t s) {
  const size_t total = count * (size_t)comm->world;
  if (comm->staging_count < total) {
    if (comm->staging) cudaFreeHost(comm->staging);
    comm->staging = nullptr;
    comm->staging_count = 0;
    NAT_CUDA_TRY(cudaHostAlloc(&comm->staging, total * sizeof(double), cudaHostAllocDefault));
    comm->staging_count = total;
  }
  double* own = comm->staging + (size_t)comm->rank * count;
  NAT_CUDA_TRY(cudaMemcpyAsync(own, buf + (size_t)comm->rank * count, count * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  const int rc = comm->host_fn(comm->host_user, comm->staging, count, comm->rank, comm->world);
  if (rc != 0) return fail(NAT_ERR_NCCL, "host all-gather callback returned %d", rc);
  // the next call's D2H into the staging buffer is stream-ordered after this copy, and the
  // host only touches the buffer again after that call's synchronisation
  NAT_CUDA_TRY(cudaMemcpyAsync(buf, comm->staging, total * sizeof(double), cudaMemcpyHostToDevice, s));
  return NAT_OK;
}
}  // namespace

// In-place all-gather of `count` doubles per rank: rank r's block lives at buf + r*count.
nat_status allgather_inplace(nat_comm* comm, double* buf, size_t count, cudaStream_t s) {
  if (comm->host_fn) return host_allgather(comm, buf, count, s);
  ncclResult_t r = ncclAllGather(buf + (size_t)comm->rank * count, buf, count, ncclDouble, comm->nccl, s);
  if (r != ncclSuccess) return fail(NAT_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  return NAT_OK;
}

nat_status allgather_inplace_many(nat_comm* comm, double* const* bufs, int nbuf, size_t count, cudaStream_t s) {
  if (comm->host_fn) {
    for (int q = 0; q < nbuf; ++q) {
      nat_status st = host_allgather(comm, bufs[q], count, s);
      if (st != NAT_OK) return st;
    }
    return NAT_OK;
  }
  ncclResult_t r = ncclGroupStart();
  for (int q = 0; q < nbuf && r == ncclSuccess; ++q)
    r = ncclAllGather(bufs[q] + (size_t)comm->rank * count, bufs[q], count, ncclDouble, comm->nccl, s);
  const ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess) return fail(NAT_ERR_NCCL, "ncclAllGather (group): %s", ncclGetErrorString(r));
  if (r2 != ncclSuccess) return fail(NAT_ERR_NCCL, "ncclGroupEnd: %s", ncclGetErrorString(r2));
  return NAT_OK;
}
}  // namespace nat
