// NCCL communicator for the row-sharded GMRES (NVLink 5 / NVSwitch inside one box).
// Rank 0 creates the ncclUniqueId; the caller broadcasts its 128 bytes with
// torch.distributed and every rank builds its own communicator from it.
#include <nccl.h>

#include <cstring>

#include "nat_comm.cuh"
#include "nat_internal.cuh"

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");

extern "C" nat_status nat_comm_unique_id(uint8_t* id) {
  NAT_REQUIRE(id, "id must be a host buffer of 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nat::fail(NAT_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(id, &u, sizeof u);
  return NAT_OK;
}

extern "C" nat_status nat_comm_create_from_id(nat_comm** comm, const uint8_t* id, int rank, int world) {
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

extern "C" nat_status nat_comm_destroy(nat_comm* comm) {
  if (!comm) return NAT_OK;
  ncclResult_t r = (comm->borrowed || !comm->nccl) ? ncclSuccess : ncclCommDestroy(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return nat::fail(NAT_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return NAT_OK;
}

namespace nat {
// In-place all-gather of `count` doubles per rank: rank r's block lives at buf + r*count.
nat_status allgather_inplace(nat_comm* comm, double* buf, size_t count, cudaStream_t s) {
  ncclResult_t r = ncclAllGather(buf + (size_t)comm->rank * count, buf, count, ncclDouble, comm->nccl, s);
  if (r != ncclSuccess) return fail(NAT_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  return NAT_OK;
}
}  // namespace nat
