// Internal radiation entry shared by nat_radiate_field and the MC operators.
#pragma once
#include "nat_internal.cuh"

namespace nat {

struct RadInput {
  int64_t n_src;
  const double* xyz;  // [3][n_src]
  const double* nrm;  // [3][n_src]
  const double* w;    // [n_src] or nullptr => w_const
  double w_const;
  int n_modes;
  const double2* p;   // [n_modes][ldpg] or nullptr (=> 0)
  const double2* g;   // [n_modes][ldpg] or nullptr (=> 0)
  int64_t ldpg;
  double center[3];
  float self_r2;      // self mode: pairs with fp32 r^2 <= self_r2 are skipped (0 => self pair only)
  const unsigned long long* skip = nullptr;  // device word; when it reads 0 the launches return at once
                                             // (Krylov driver: every system has converged)
  int64_t plan_lis = 0;  // > 0: choose the launch shape (targets per thread, source chunks) for
                         // this many targets instead of n_lis — a row block of a row-sharded
                         // operator then sums every row in the same order as the full operator
};

size_t radiate_ws_bytes(nat_prec prec, int64_t n_src, int n_modes, int64_t n_lis, int kind = 0,
                        int64_t plan_lis = 0);
// Largest workspace over 1..max_modes wavenumbers (callers that shrink the mode set).
size_t radiate_ws_bytes_upto(nat_prec prec, int64_t n_src, int max_modes, int64_t n_lis);
// out[m][l] (c128 [n_modes][n_lis]) = sum_s w_s [p_ms dG_m/dn_y - g_ms G_m](x_l, y_s);
// self = true excludes the pair with identical coordinates (targets == sources).
// Split-K partials left unreduced for a fused caller epilogue: part[split][mode][lis].
struct RadPartials {
  const double2* part = nullptr;
  int n_split = 0;
};
nat_status radiate_internal(const RadInput& in, nat_prec prec, const double* k, int64_t n_lis,
                            const double* lis, double2* out, void* ws, size_t ws_bytes, bool self,
                            cudaStream_t s, RadPartials* keep = nullptr);

}  // namespace nat
