// Batched, deterministic GMRES engine (row a7; reading R-gmres).
// Up to 64 systems iterate in lockstep.  Everything runs on the device: CGS2 Arnoldi,
// the Givens update of the Hessenberg columns, the convergence test and the final
// back-substitution.  The host only enqueues iterations, one ahead of the convergence
// mask it has read back, so the GPU never waits for the host between iterations; an
// iteration enqueued after every system converged returns at once in every kernel.
#pragma once
#include <functional>
#include <vector>

#include "nat_internal.cuh"

namespace nat {

struct DevSys {
  double beta;  // ||b||
  int k;        // Arnoldi steps taken
  int flags;    // kSysConverged | kSysNonFinite
};
constexpr int kSysConverged = 1;
constexpr int kSysNonFinite = 2;

struct KrylovWs {
  double2* V;     // [(m+1)][nsys][ldv] Arnoldi basis
  double2* W;     // [m][nsys][ldv] operator products A V_j (final residual by linearity)
  float2* Vf;     // [(m+1)][nsys][ldv] the basis in fp32 (fp32 solves, reading R-basis32)
  double2* w;     // [nsys][ldv]
  double2* part;  // [nsys][m+1][nchunk]
  double2* h;     // [nsys][m+2]  current Arnoldi column
  double2* h2;    // [nsys][m+2]
  double2* y;     // [nsys][m]
  double2* npart; // [nsys][ceil(n/256)] norm partials
  double2* H;     // [nsys][m][m+1] rotated Hessenberg columns
  double2* cs;    // [nsys][m] Givens cosines
  double2* sn;    // [nsys][m] Givens sines
  double2* gam;   // [nsys][m+1] rotated residual vector
  DevSys* sys;    // [nsys]
  unsigned long long* mask;  // [1] systems still iterating
  unsigned* cnt;  // [2][64] + 1 last-block counters (zeroed at the start of every solve)
};

constexpr int kKrylovChunk = 1024;

size_t krylov_workspace(int nsys, int64_t n, int64_t ldv, int max_iter, Carver& c, KrylovWs* w);

// Operator: out[s] = A_s in[s] for every system s with (active >> s) & 1; in/out are
// [nsys][ldv] c128 arrays.  `active` is the host's view (possibly one iteration stale);
// `dmask` (device, may be null) is the live mask: an operator may return at once when
// it reads 0.  Must enqueue on `s` and return NAT_OK or an error.
using KrylovOp = std::function<nat_status(const double2* in, double2* out, uint64_t active,
                                          const unsigned long long* dmask, cudaStream_t s)>;

struct KrylovResult {
  int iters, converged;
  double rel_residual;
};

// Solves A_s x_s = b_s (b, x: [nsys][ldv]; only the first n entries of each row used).
nat_status gmres_batched(int nsys, int64_t n, int64_t ldv, const double2* b, double2* x,
                         const KrylovOp& op, double tol, int max_iter, const KrylovWs& ws,
                         std::vector<KrylovResult>& res, cudaStream_t s, double* t_op_s = nullptr,
                         bool basis32 = false);

// Reusable timing events of the calling thread on the current device (pool `slot`).
cudaEvent_t timing_event(int slot, size_t i);

}  // namespace nat
