// Batched, deterministic GMRES engine (row a7; reading R-gmres).
// Up to 64 systems iterate in lockstep; each has its own Hessenberg/Givens state on the
// host (O(m) scalars per iteration), every vector operation runs in CUDA kernels with a
// fixed reduction order (results do not depend on the number of GPUs).
#pragma once
#include <functional>
#include <vector>

#include "nat_internal.cuh"

namespace nat {

struct KrylovWs {
  double2* V;     // [(m+1)][nsys][ldv]
  double2* w;     // [nsys][ldv]
  double2* part;  // [nsys][m+1][nchunk]
  double2* h;     // [nsys][m+2]
  double2* h2;    // [nsys][m+2]
  double2* y;     // [nsys][m]
  double2* npart; // [nsys][ceil(n/256)] norm partials
  unsigned* cnt;  // [2][64] last-block counters (zeroed at the start of every solve)
};

constexpr int kKrylovChunk = 4096;

size_t krylov_workspace(int nsys, int64_t n, int64_t ldv, int max_iter, Carver& c, KrylovWs* w);

// Operator: out[s] = A_s in[s] for every system s with (active >> s) & 1; in/out are
// [nsys][ldv] c128 arrays.  Must enqueue on `s` and return NAT_OK or an error.
using KrylovOp = std::function<nat_status(const double2* in, double2* out, uint64_t active, cudaStream_t s)>;

struct KrylovResult {
  int iters, converged;
  double rel_residual;
};

// Solves A_s x_s = b_s (b, x: [nsys][ldv]; only the first n entries of each row used).
nat_status gmres_batched(int nsys, int64_t n, int64_t ldv, const double2* b, double2* x,
                         const KrylovOp& op, double tol, int max_iter, const KrylovWs& ws,
                         std::vector<KrylovResult>& res, cudaStream_t s, double* t_op_s = nullptr);

}  // namespace nat
