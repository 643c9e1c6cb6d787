// Rows a4 + a5 — dense collocation assembly of the conventional BIE and a6 — the
// stored-matrix matvec.
//
// Equation: Eq. BM with beta = 0 ("i.e., beta = 0" P:191), outward normals
// (reading R-sign): 1/2 p(x) - int p dG/dn_y = - int g G.  P0 collocation at centroids
// (reading R-colloc): A = 1/2 I - K, b = -V g,
//   K_ij = int_{T_j} dG/dn_y(c_i, y) dS,  V_ij = int_{T_j} G(c_i, y) dS.
// Quadrature by pair class ("adjacent or identical elements"): far rule on every
// pair (a4, fused with the row reduction of b so V is never stored), then the near and
// self kernels (a5) overwrite the near entries of A and correct b in a fixed order.
//
// B200 mapping: far kernel CTA = 16 rows x 1024 columns, one column per
// thread per pass (its 3 quadrature points, weights and normal in registers), the
// 16 collocation points broadcast from shared memory; every warp stores 32 consecutive
// entries of a row (coalesced 256 B / 512 B); the RHS partial sums stay in registers
// and are reduced once per CTA (warp shuffles, then a fixed-order shared-memory sum).
// Near pairs: one 32-lane group per vertex-sharing pair (448 points), one 8-lane group
// per close pair (28 points), fp64 point positions and differences, kernel math in the
// path's precision.  Self term: one thread per row, polar Gauss-Legendre in fp64.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "f32x2.cuh"
#include "nat_internal.cuh"
#include "pair.cuh"

namespace {
namespace cg = cooperative_groups;

using nat::C2;

constexpr int kThreads = 256;
#ifndef NAT_FAR_TI
#define NAT_FAR_TI 16          // rows per far CTA (tuning)
#endif
constexpr int kTI = NAT_FAR_TI;  // rows per far CTA
#ifndef NAT_FAR_UNROLL
#define NAT_FAR_UNROLL 1       // column passes interleaved by the packed far kernel (tuning)
#endif
constexpr int kFarUnroll = NAT_FAR_UNROLL;
#ifndef NAT_FAR_MINB
#define NAT_FAR_MINB 2         // resident CTAs per SM the packed far kernel is compiled for (tuning)
#endif
constexpr int kFarMinBlocks = NAT_FAR_MINB;
constexpr int kTI64 = 4;      // rows per CTA of the fp64 far kernel (16 unrolled fp64 rows -> 238
                              // registers, 8 warps/SM; ncu r01 matrix-free C5 capture)
#ifndef NAT_FAR_CC
#define NAT_FAR_CC 16          // column passes per far CTA (tuning; A/B profiles/r01_ab_far_cc.txt)
#endif
constexpr int kCC = NAT_FAR_CC;  // column passes per far CTA (columns = 256 * kCC)
constexpr int kMaxFarQ = 7;
constexpr int kNRmax = 2;

// ------------------------------------------------------------------------------------
// quadrature tables (the library's own host code; DESIGN.md §3 R-colloc / R-self)
// ------------------------------------------------------------------------------------
struct Pt {
  double l1, l2, l3, w;
};

// The 1- and 7-point far rules contain the centroid, i.e. the collocation point of the row's
// own triangle: their far-rule self pair is singular and is zeroed by the far kernels.
template <int NQ>
constexpr bool kCentroidRule = (NQ == 1 || NQ == 7);

bool base_rule(int npts, std::vector<Pt>& out) {
  out.clear();
  if (npts == 1) {
    out.push_back({1.0 / 3, 1.0 / 3, 1.0 / 3, 1.0});
  } else if (npts == 3) {
    const double a = 2.0 / 3, b = 1.0 / 6;
    out = {{a, b, b, 1.0 / 3}, {b, a, b, 1.0 / 3}, {b, b, a, 1.0 / 3}};
  } else if (npts == 6) {  // Dunavant degree 4
    const double a1 = 0.10810301816807023, b1 = 0.44594849091596489, w1 = 0.22338158967801147;
    const double a2 = 0.81684757298045851, b2 = 0.091576213509770743, w2 = 0.10995174365532187;
    out = {{a1, b1, b1, w1}, {b1, a1, b1, w1}, {b1, b1, a1, w1},
           {a2, b2, b2, w2}, {b2, a2, b2, w2}, {b2, b2, a2, w2}};
  } else if (npts == 7) {  // Radon degree 5
    const double s15 = std::sqrt(15.0);
    const double ap = (6 + s15) / 21, am = (6 - s15) / 21;
    const double wp = (155 + s15) / 1200, wm = (155 - s15) / 1200;
    out.push_back({1.0 / 3, 1.0 / 3, 1.0 / 3, 9.0 / 40});
    for (int s = 0; s < 2; ++s) {
      double a = s == 0 ? ap : am, w = s == 0 ? wp : wm, b = 1 - 2 * a;
      out.push_back({b, a, a, w});
      out.push_back({a, b, a, w});
      out.push_back({a, a, b, w});
    }
  } else {
    return false;
  }
  return true;
}

struct Bary {
  double p[3][3];
};

void subdivide(const Bary& t, int level, std::vector<Bary>& out) {
  if (level == 0) {
    out.push_back(t);
    return;
  }
  Bary c[4];
  double m12[3], m13[3], m23[3];
  for (int a = 0; a < 3; ++a) {
    m12[a] = (t.p[0][a] + t.p[1][a]) / 2;
    m13[a] = (t.p[0][a] + t.p[2][a]) / 2;
    m23[a] = (t.p[1][a] + t.p[2][a]) / 2;
  }
  for (int a = 0; a < 3; ++a) {
    c[0].p[0][a] = t.p[0][a]; c[0].p[1][a] = m12[a];    c[0].p[2][a] = m13[a];
    c[1].p[0][a] = m12[a];    c[1].p[1][a] = t.p[1][a]; c[1].p[2][a] = m23[a];
    c[2].p[0][a] = m13[a];    c[2].p[1][a] = m23[a];    c[2].p[2][a] = t.p[2][a];
    c[3].p[0][a] = m12[a];    c[3].p[1][a] = m23[a];    c[3].p[2][a] = m13[a];
  }
  for (auto& ch : c) subdivide(ch, level - 1, out);
}

void composite_rule(int level, std::vector<Pt>& out) {
  std::vector<Pt> base;
  base_rule(7, base);
  std::vector<Bary> subs;
  Bary root{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
  subdivide(root, level, subs);
  out.clear();
  const double scale = 1.0 / (double)subs.size();
  for (auto& s : subs)
    for (auto& q : base) {
      Pt p;
      double l[3];
      for (int a = 0; a < 3; ++a) l[a] = q.l1 * s.p[0][a] + q.l2 * s.p[1][a] + q.l3 * s.p[2][a];
      p.l1 = l[0];
      p.l2 = l[1];
      p.l3 = l[2];
      p.w = q.w * scale;
      out.push_back(p);
    }
}

// Gauss-Legendre nodes/weights on [-1, 1] by Newton iteration on P_n.
void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(nat::kPi * (i + 0.75) / (n + 0.5)), pp = 0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1, p2 = 0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1);
      double dz = p1 / pp;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    x[i] = -z;
    x[n - 1 - i] = z;
    w[i] = w[n - 1 - i] = 2.0 / ((1 - z * z) * pp * pp);
  }
}

struct Opts {
  int far_pts, lev_S, lev_N, gl;
  double eta;
  bool bm;  // Burton-Miller (NEXT-1, reading R-bm)
  bool gal = false;  // Galerkin (NEXT-2, reading R-galerkin)
  int ss = 4;        // Sauter-Schwab order
};

Opts opts_of(const nat_quad_opts* o) {
  Opts r{3, 3, 1, 16, 4.0, false};
  if (o) {
    r.bm = o->burton_miller != 0;
    if (o->far_pts) r.far_pts = o->far_pts;
    if (o->near_levels_S) r.lev_S = o->near_levels_S;
    if (o->near_levels_N) r.lev_N = o->near_levels_N;
    if (o->self_theta_pts) r.gl = o->self_theta_pts;
    if (o->near_eta > 0) r.eta = o->near_eta;
    r.gal = o->galerkin != 0;
    if (o->ss_order) r.ss = o->ss_order;
  }
  return r;
}

// ------------------------------------------------------------------------------------
// kernels
// ------------------------------------------------------------------------------------
template <typename R>
struct FarCols {        // per column j: NQ points (relative to centre), weights, normal
  const R* qxyz;        // [NQ][3][n]
  const R* qw;          // [NQ][n]  (omega_q A_j / 4pi)
  const R* nrm;         // [3][n]
};

template <typename R>
__global__ void far_prep_kernel(int64_t nv, int64_t n, const double* __restrict__ vx,
                                const int32_t* __restrict__ tri, const double* __restrict__ nrm,
                                const double* __restrict__ area, const double4* __restrict__ rule,
                                int NQ, double cx, double cy, double cz, R* __restrict__ qxyz,
                                R* __restrict__ qw, R* __restrict__ nout) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int a = tri[j], b = tri[n + j], c = tri[2 * n + j];
  const double cen[3] = {cx, cy, cz};
  for (int q = 0; q < NQ; ++q) {
    double4 L = rule[q];
    for (int d = 0; d < 3; ++d) {
      const double* X = vx + d * nv;
      double y = (L.x * X[a] + L.y * X[b]) + L.z * X[c];
      qxyz[((size_t)q * 3 + d) * n + j] = (R)(y - cen[d]);
    }
    qw[(size_t)q * n + j] = (R)(L.w * area[j] * nat::kInv4Pi);
  }
  for (int d = 0; d < 3; ++d) nout[(size_t)d * n + j] = (R)nrm[(size_t)d * n + j];
}

template <typename R, int NQ>
__device__ __forceinline__ void far_entry(const R (&y)[NQ][3], const R (&w)[NQ], R nx, R ny, R nz,
                                          R cx, R cy, R cz, R k, R& Vr, R& Vi, R& Kr, R& Ki) {
  Vr = Vi = Kr = Ki = R(0);
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    nat::pair_accumulate<R>(y[q][0] - cx, y[q][1] - cy, y[q][2] - cz, nx, ny, nz, w[q], k, Vr, Vi,
                            Kr, Ki);
}

// Far-rule RHS operator entry of Burton-Miller: (V + beta K')_ij with beta = i/k, i.e.
// (V.x - K'.y / k, V.y + K'.x / k); m = the target's normal n_x.
template <typename R, int NQ>
__device__ __forceinline__ void far_entry_bm_rhs(const R (&y)[NQ][3], const R (&w)[NQ], R nx, R ny, R nz, R mx,
                                                 R my, R mz, R cx, R cy, R cz, R k, R& Br, R& Bi) {
  nat::C2<R> V{R(0), R(0)}, K{R(0), R(0)}, Kp{R(0), R(0)}, W{R(0), R(0)};
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    nat::pair_accumulate_bm<R>(y[q][0] - cx, y[q][1] - cy, y[q][2] - cz, nx, ny, nz, mx, my, mz, w[q], k, V, K,
                               Kp, W);
  Br = V.x - Kp.y / k;
  Bi = V.y + Kp.x / k;
}

template <typename R>
__device__ __forceinline__ void store_entry(void* A, size_t idx, R re, R im) {
  if constexpr (sizeof(R) == 4)
    reinterpret_cast<float2*>(A)[idx] = make_float2(re, im);
  else
    reinterpret_cast<double2*>(A)[idx] = make_double2(re, im);
}

template <typename R>
struct FarArgs {
  int64_t n, row_begin, rows, lda;
  FarCols<R> cols;
  const double* cen;     // geom centroid [3][n]
  const double* nrm;     // geom normal [3][n] (Burton-Miller: the rows' n_x)
  double cx, cy, cz;
  R k;
  int n_rhs, rhs0;       // this pass covers rhs [rhs0, rhs0 + NR)
  const double2* g;      // [n_rhs][n]
  void* A;
  bool store_A;
  double2* bpart;        // [n_colblk][n_rhs][rows]
  const unsigned long long* skip;  // MV (matrix-free operator inside GMRES): return when *skip == 0
  // Galerkin (NEXT-2, NTQ > 1 test points per row): row triangles' vertices and areas,
  // the test rule (the far rule, barycentric + weight)
  const double* vx;
  const int32_t* tri;
  int64_t nv;
  const double* area;
  const double4* rule;
};

// Row test points of the far kernels, relative to the centre (cx, cy, cz): NTQ = 1 is the
// centroid (collocation, weight 1); NTQ > 1 the far rule on T_i with weights w_t |T_i|
// (Galerkin, reading R-galerkin).
template <typename R, int NTQ>
__device__ __forceinline__ void row_points(const FarArgs<R>& a, int64_t i, double (&c)[NTQ][3], double (&wt)[NTQ]) {
  const int64_t n = a.n;
  if constexpr (NTQ == 1) {
    c[0][0] = a.cen[i] - a.cx;
    c[0][1] = a.cen[n + i] - a.cy;
    c[0][2] = a.cen[2 * n + i] - a.cz;
    wt[0] = 1.0;
  } else {
    double v[3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const int vi = a.tri[p * n + i];
#pragma unroll
      for (int d = 0; d < 3; ++d) v[p][d] = a.vx[d * a.nv + vi];
    }
    const double cen[3] = {a.cx, a.cy, a.cz};
#pragma unroll
    for (int t = 0; t < NTQ; ++t) {
      const double4 L = a.rule[t];
#pragma unroll
      for (int d = 0; d < 3; ++d) c[t][d] = ((L.x * v[0][d] + L.y * v[1][d]) + L.z * v[2][d]) - cen[d];
      wt[t] = L.w * a.area[i];
    }
  }
}

// Generic far assembly (fp64, and fp32 Burton-Miller).  BM: A_ij = -K_ij - beta W_ij and
// the RHS operator V + beta K' (beta = i/k, reading R-bm).
// MV (matrix-free matvec, NEXT-3): NR = 1, g = the iterate x; accumulates (A^far x)_i =
// sum_j (-K_ij) x_j over the CTA's columns instead of storing A (bpart gets +sum).
// NTQ > 1 (Galerkin, NEXT-2): each entry sums NTQ test points of T_i with weights
// w_t |T_i|; the diagonal j == i is left to the Sauter-Schwab self kernel (0 here).
template <typename R, int NQ, int NR, bool BM = false, bool MV = false, int TI = kTI, int NTQ = 1>
__global__ void __launch_bounds__(kThreads) far_kernel(FarArgs<R> a) {
  static_assert(!MV || (NR == 1 && !BM), "matrix-free: one iterate, conventional BIE");
  static_assert(NTQ == 1 || (!BM && !MV), "Galerkin: conventional BIE, stored operator");
  if (MV && a.skip && *a.skip == 0ull) return;
  __shared__ R s_c[NTQ][3][TI];
  __shared__ R s_wt[NTQ][TI];
  __shared__ R s_m[3][TI];  // BM: row normals
  __shared__ double2 s_red[kThreads / 32][TI][NR > 0 ? NR : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.y * TI;
  const int64_t n = a.n;
  if (tid < TI) {
    int64_t r = i0 + tid;
    int64_t i = a.row_begin + (r < a.rows ? r : 0);
    double c[NTQ][3], wt[NTQ];
    row_points<R, NTQ>(a, i, c, wt);
#pragma unroll
    for (int t = 0; t < NTQ; ++t) {
      s_c[t][0][tid] = (R)c[t][0];
      s_c[t][1][tid] = (R)c[t][1];
      s_c[t][2][tid] = (R)c[t][2];
      s_wt[t][tid] = (R)wt[t];
    }
    if constexpr (BM) {
      s_m[0][tid] = (R)a.nrm[i];
      s_m[1][tid] = (R)a.nrm[n + i];
      s_m[2][tid] = (R)a.nrm[2 * n + i];
    }
  }
  __syncthreads();
  const int nrows = (int)nat::min64(TI, a.rows - i0);
  C2<R> bacc[TI][NR > 0 ? NR : 1];
#pragma unroll
  for (int t = 0; t < TI; ++t)
#pragma unroll
    for (int q = 0; q < (NR > 0 ? NR : 1); ++q) bacc[t][q] = {R(0), R(0)};

  for (int cc = 0; cc < kCC; ++cc) {
    const int64_t j = (int64_t)blockIdx.x * (kThreads * kCC) + cc * kThreads + tid;
    const bool valid = j < n;
    const int64_t jj = valid ? j : 0;
    R y[NQ][3], w[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      y[q][0] = a.cols.qxyz[((size_t)q * 3 + 0) * n + jj];
      y[q][1] = a.cols.qxyz[((size_t)q * 3 + 1) * n + jj];
      y[q][2] = a.cols.qxyz[((size_t)q * 3 + 2) * n + jj];
      w[q] = valid ? a.cols.qw[(size_t)q * n + jj] : R(0);
    }
    const R nx = a.cols.nrm[jj], ny = a.cols.nrm[n + jj], nz = a.cols.nrm[2 * n + jj];
    C2<R> gj[NR > 0 ? NR : 1];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      double2 gv = valid ? a.g[(size_t)(a.rhs0 + q) * n + jj] : make_double2(0.0, 0.0);
      gj[q] = {(R)gv.x, (R)gv.y};
    }
#pragma unroll
    for (int t = 0; t < TI; ++t) {
      if (t < nrows) {
        R Vr, Vi, Kr, Ki;
        if constexpr (BM) {
          C2<R> V{R(0), R(0)}, K{R(0), R(0)}, Kp{R(0), R(0)}, W{R(0), R(0)};
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            nat::pair_accumulate_bm<R>(y[q][0] - s_c[0][0][t], y[q][1] - s_c[0][1][t], y[q][2] - s_c[0][2][t], nx, ny, nz,
                                       s_m[0][t], s_m[1][t], s_m[2][t], w[q], a.k, V, K, Kp, W);
          // A = -K - (i/k) W;  RHS operator V + (i/k) K'
          Kr = K.x - W.y / a.k;
          Ki = K.y + W.x / a.k;
          Vr = V.x - Kp.y / a.k;
          Vi = V.y + Kp.x / a.k;
        } else if constexpr (NTQ == 1) {
          far_entry<R, NQ>(y, w, nx, ny, nz, s_c[0][0][t], s_c[0][1][t], s_c[0][2][t], a.k, Vr, Vi, Kr, Ki);
        } else {
          Vr = Vi = Kr = Ki = R(0);
#pragma unroll
          for (int tq = 0; tq < NTQ; ++tq) {
            R vr, vi, kr, ki;
            far_entry<R, NQ>(y, w, nx, ny, nz, s_c[tq][0][t], s_c[tq][1][t], s_c[tq][2][t], a.k, vr, vi, kr, ki);
            const R wt = s_wt[tq][t];
            Vr += wt * vr;
            Vi += wt * vi;
            Kr += wt * kr;
            Ki += wt * ki;
          }
          // self pair (Sauter-Schwab kernel) and padding columns (jj = 0 may be the row)
          if (!valid || j == a.row_begin + i0 + t) Vr = Vi = Kr = Ki = R(0);
        }
        if constexpr (NTQ == 1 && kCentroidRule<NQ>) {
          // the 1- and 7-point rules contain the centroid = the collocation point: the self
          // pair is singular under the far rule; it is zeroed (the self kernel adds the exact
          // value and subtracts nothing) — a select, NaN-safe
          if (!valid || j == a.row_begin + i0 + t) Vr = Vi = Kr = Ki = R(0);
        }
        if (!MV && a.store_A && valid) store_entry<R>(a.A, (size_t)(i0 + t) * a.lda + j, -Kr, -Ki);
        if constexpr (MV) {  // (-K) x_j
          bacc[t][0].x -= Kr * gj[0].x - Ki * gj[0].y;
          bacc[t][0].y -= Kr * gj[0].y + Ki * gj[0].x;
        } else {
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            bacc[t][q].x += Vr * gj[q].x - Vi * gj[q].y;
            bacc[t][q].y += Vr * gj[q].y + Vi * gj[q].x;
          }
        }
      }
    }
  }
  if constexpr (NR > 0) {
#pragma unroll
    for (int t = 0; t < TI; ++t)
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        double vx = (double)bacc[t][q].x, vy = (double)bacc[t][q].y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          vx += __shfl_xor_sync(0xffffffffu, vx, o);
          vy += __shfl_xor_sync(0xffffffffu, vy, o);
        }
        if (lane == 0) s_red[warp][t][q] = make_double2(vx, vy);
      }
    __syncthreads();
    if (tid < TI * NR) {
      const int t = tid / NR, q = tid % NR;
      if (t < nrows) {
        double2 s = s_red[0][t][q];
        for (int wv = 1; wv < kThreads / 32; ++wv) {
          s.x += s_red[wv][t][q].x;
          s.y += s_red[wv][t][q].y;
        }
        // b = -V g  (MV: + sum_j A^far_ij x_j)
        a.bpart[((size_t)blockIdx.x * a.n_rhs + a.rhs0 + q) * a.rows + i0 + t] =
            MV ? s : make_double2(-s.x, -s.y);
      }
    }
  }
}

// NAT_FP32 far assembly on the packed FP32x2 pipe: two rows (collocation points) share
// each instruction, the column's quadrature data is broadcast into both halves.  Per
// quadrature point and row: 11 packed-pipe instructions + 1 FMUL.RZ + 3 MUFU.  The kernel
// accumulates -K directly (A_ij = -K_ij off the diagonal) and V g for the RHS.
// MV (matrix-free matvec, NEXT-3): NR = 1 and g = the iterate x; the row sums are
// sum_j (-K_ij) x_j = (A^far x)_i (no store, V unused).
// NTQ > 1 (Galerkin, NEXT-2): NTQ test points per row with weights w_t |T_i| (staged in
// shared memory); the self pair and padding columns are zeroed (Sauter-Schwab self kernel).
template <int NQ, int NR, bool MV = false, int NTQ = 1>
__global__ void __launch_bounds__(kThreads, kFarMinBlocks) far_kernel_x2(FarArgs<float> a) {
  static_assert(kTI % 2 == 0, "row pairs");
  static_assert(!MV || NR == 1, "matrix-free: one iterate");
  static_assert(NTQ == 1 || !MV, "Galerkin: stored operator");
  if (MV && a.skip && *a.skip == 0ull) return;
  constexpr int TP = kTI / 2;
  constexpr int NRr = NR > 0 ? NR : 1;
  __shared__ __align__(16) f2r s_c[NTQ][3][TP];
  __shared__ __align__(16) f2r s_wt[NTQ][TP];
  __shared__ double2 s_red[kThreads / 32][kTI][NRr];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.y * kTI;
  const int64_t n = a.n;
  if (tid < TP) {
    double c[2][NTQ][3], wt[2][NTQ];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = i0 + 2 * tid + h;
      const int64_t i = a.row_begin + (r < a.rows ? r : 0);
      row_points<float, NTQ>(a, i, c[h], wt[h]);
    }
#pragma unroll
    for (int t = 0; t < NTQ; ++t) {
#pragma unroll
      for (int d = 0; d < 3; ++d) s_c[t][d][tid] = f2pack((float)c[0][t][d], (float)c[1][t][d]);
      s_wt[t][tid] = f2pack((float)wt[0][t], (float)wt[1][t]);
    }
  }
  __syncthreads();
  const int nrows = (int)nat::min64(kTI, a.rows - i0);
  const f2r kk = f2pack(a.k, a.k), nkk = f2pack(-a.k, -a.k);
  f2r br[TP][NRr], bi[TP][NRr];  // sum_j V_ij g_j for the row pair (real / imaginary)
#pragma unroll
  for (int t = 0; t < TP; ++t)
#pragma unroll
    for (int q = 0; q < NRr; ++q) br[t][q] = bi[t][q] = 0ull;

  // full row blocks (all but the last) run without per-row guards, so the row pairs of a
  // column form one straight-line block the scheduler can interleave
  auto columns = [&](auto full_tag) {
    constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll kFarUnroll
    for (int cc = 0; cc < kCC; ++cc) {
      const int64_t j = (int64_t)blockIdx.x * (kThreads * kCC) + cc * kThreads + tid;
      const bool valid = j < n;
      const int64_t jj = valid ? j : 0;
      f2r y[NQ][3], w[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float v = a.cols.qxyz[((size_t)q * 3 + d) * n + jj];
          y[q][d] = f2pack(v, v);
        }
        const float wv = valid ? a.cols.qw[(size_t)q * n + jj] : 0.f;
        w[q] = f2pack(wv, wv);
      }
      const float nxs = a.cols.nrm[jj], nys = a.cols.nrm[n + jj], nzs = a.cols.nrm[2 * n + jj];
      const f2r nx = f2pack(nxs, nxs), ny = f2pack(nys, nys), nz = f2pack(nzs, nzs);
      // d.n = y_q.n - c.n: the column part once per column, the row part once per row pair
      f2r yn[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float v = fmaf(f2lo(y[q][2]), nzs, fmaf(f2lo(y[q][1]), nys, f2lo(y[q][0]) * nxs));
        yn[q] = f2pack(v, v);
      }
      f2r gr[NRr], gi[NRr], ngi[NRr];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const double2 gv = valid ? a.g[(size_t)(a.rhs0 + q) * n + jj] : make_double2(0.0, 0.0);
        gr[q] = f2pack((float)gv.x, (float)gv.x);
        gi[q] = f2pack((float)gv.y, (float)gv.y);
        ngi[q] = f2pack(-(float)gv.y, -(float)gv.y);
      }
      // running pointer to A[i0 + 2t][j] (one 64-bit add per row pair instead of a
      // 64-bit multiply per store)
      float2* arow = reinterpret_cast<float2*>(a.A) + (size_t)i0 * a.lda + jj;
      const int64_t ld = a.lda;
#pragma unroll
      for (int t = 0; t < TP; ++t, arow += 2 * ld) {
        if (FULL || 2 * t < nrows) {
          f2r Vr = 0ull, Vi = 0ull, Kr = 0ull, Ki = 0ull;  // K here is -K
#pragma unroll
          for (int tq = 0; tq < NTQ; ++tq) {
          const f2r cx = s_c[tq][0][t], cy = s_c[tq][1][t], cz = s_c[tq][2][t];
          const f2r cn = f2fma(cz, nz, f2fma(cy, ny, f2mul(cx, nx)));
          f2r vr = 0ull, vi = 0ull, kr_ = 0ull, ki_ = 0ull;
          f2r& Vr_ = NTQ == 1 ? Vr : vr;
          f2r& Vi_ = NTQ == 1 ? Vi : vi;
          f2r& Kr_ = NTQ == 1 ? Kr : kr_;
          f2r& Ki_ = NTQ == 1 ? Ki : ki_;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const f2r dx = f2sub(y[q][0], cx), dy = f2sub(y[q][1], cy), dz = f2sub(y[q][2], cz);
            const f2r r2 = f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx)));
            const f2r dn = f2sub(yn[q], cn);
            const f2r rho = f2pack(nat::pair_rsqrt(f2lo(r2)), nat::pair_rsqrt(f2hi(r2)));
            const f2r rr = f2mul(r2, rho);
            const f2r kr = f2mul(rr, kk), nkr = f2mul(rr, nkk);
            float s0, c0, s1, c1;
            __sincosf(f2lo(kr), &s0, &c0);
            __sincosf(f2hi(kr), &s1, &c1);
            const f2r sn = f2pack(s0, s1), cs = f2pack(c0, c1);
            const f2r tw = f2mul(w[q], rho);               // w G-part: tw e^{ikr}
            Vr_ = f2fma(tw, cs, Vr_);
            Vi_ = f2fma(tw, sn, Vi_);
            const f2r u = f2mul(tw, f2mul(dn, f2mul(rho, rho)));
            // -K += u (c + kr s) + i u (s - kr c)   [K = u (ikr - 1) e^{ikr}]
            Kr_ = f2fma(u, f2fma(kr, sn, cs), Kr_);
            Ki_ = f2fma(u, f2fma(nkr, cs, sn), Ki_);
          }
          if constexpr (NTQ > 1) {  // test weight w_t |T_i|
            const f2r wt = s_wt[tq][t];
            Vr = f2fma(wt, vr, Vr);
            Vi = f2fma(wt, vi, Vi);
            Kr = f2fma(wt, kr_, Kr);
            Ki = f2fma(wt, ki_, Ki);
          }
          }
          if constexpr (NTQ > 1 || kCentroidRule<NQ>) {  // self pair and padding columns -> 0 (select, NaN-safe)
            const int64_t ri = a.row_begin + i0 + 2 * t;
            const bool z0 = !valid || j == ri, z1 = !valid || j == ri + 1;
            if (z0 || z1) {
              Vr = f2pack(z0 ? 0.f : f2lo(Vr), z1 ? 0.f : f2hi(Vr));
              Vi = f2pack(z0 ? 0.f : f2lo(Vi), z1 ? 0.f : f2hi(Vi));
              Kr = f2pack(z0 ? 0.f : f2lo(Kr), z1 ? 0.f : f2hi(Kr));
              Ki = f2pack(z0 ? 0.f : f2lo(Ki), z1 ? 0.f : f2hi(Ki));
            }
          }
          if (!MV && a.store_A && valid) {
            arow[0] = make_float2(f2lo(Kr), f2lo(Ki));
            if (FULL || 2 * t + 1 < nrows) arow[ld] = make_float2(f2hi(Kr), f2hi(Ki));
          }
          if constexpr (MV) {  // (-K) x_j  (Kr, Ki hold -K)
            br[t][0] = f2fma(Kr, gr[0], f2fma(Ki, ngi[0], br[t][0]));
            bi[t][0] = f2fma(Kr, gi[0], f2fma(Ki, gr[0], bi[t][0]));
          } else {
#pragma unroll
            for (int q = 0; q < NR; ++q) {
              br[t][q] = f2fma(Vr, gr[q], f2fma(Vi, ngi[q], br[t][q]));
              bi[t][q] = f2fma(Vr, gi[q], f2fma(Vi, gr[q], bi[t][q]));
            }
          }
        }
      }
    }
  };
  if (nrows == kTI)
    columns(std::integral_constant<bool, true>{});
  else
    columns(std::integral_constant<bool, false>{});
  if constexpr (NR > 0) {
#pragma unroll
    for (int t = 0; t < kTI; ++t)
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const f2r pr = br[t / 2][q], pi = bi[t / 2][q];
        double vx = (double)((t & 1) ? f2hi(pr) : f2lo(pr)), vy = (double)((t & 1) ? f2hi(pi) : f2lo(pi));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          vx += __shfl_xor_sync(0xffffffffu, vx, o);
          vy += __shfl_xor_sync(0xffffffffu, vy, o);
        }
        if (lane == 0) s_red[warp][t][q] = make_double2(vx, vy);
      }
    __syncthreads();
    if (tid < kTI * NR) {
      const int t = tid / NR, q = tid % NR;
      if (t < nrows) {
        double2 s = s_red[0][t][q];
        for (int wv = 1; wv < kThreads / 32; ++wv) {
          s.x += s_red[wv][t][q].x;
          s.y += s_red[wv][t][q].y;
        }
        a.bpart[((size_t)blockIdx.x * a.n_rhs + a.rhs0 + q) * a.rows + i0 + t] =
            MV ? s : make_double2(-s.x, -s.y);
      }
    }
  }
}

// Multi-wavenumber far assembly (fp32, collocation, conventional BIE; round 2): one pass over
// the pairs forms the far entries of NK matrices A_k = -K_k (k = the NK wavenumbers of the
// call) and their right-hand-side sums V_k g, sharing per quadrature point the geometry
// (d, r^2, rsqrt, r, d.n, the weights): per pair-evaluation x wavenumber 1/NK of the shared
// work + kr, sincos and the V/K accumulation.  CTA = kTIM rows x 256 * kCC columns (the
// column blocking of the one-wavenumber kernel, so the partial-sum layout is the same).
#ifndef NAT_FAR_TIM
#define NAT_FAR_TIM 8
#endif
#ifndef NAT_FAR_MINB
#define NAT_FAR_MINB 2
#endif
constexpr int kTIM = NAT_FAR_TIM;  // rows per CTA (compile-time variants: scripts/build_variants.sh)
constexpr int kMaxK = 4;
struct FarMultiArgs {
  FarArgs<float> b;          // n, row_begin, rows, lda, cols, cen, centre, g (one RHS), rhs0 = 0
  float k[kMaxK];
  float2* A[kMaxK];          // c64 [rows][lda]
  double2* bpart[kMaxK];     // [n_colblk][1][rows]
};

template <int NQ, int NK>
__global__ void __launch_bounds__(kThreads, NAT_FAR_MINB) far_kernel_multi(FarMultiArgs m) {
  constexpr int TP = kTIM / 2;
  const FarArgs<float>& a = m.b;
  __shared__ __align__(16) f2r s_c[3][TP];
  __shared__ double2 s_red[kThreads / 32][kTIM][NK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.y * kTIM;
  const int64_t n = a.n;
  if (tid < TP) {
    double c[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = i0 + 2 * tid + h;
      const int64_t i = a.row_begin + (r < a.rows ? r : 0);
      c[h][0] = a.cen[i] - a.cx;
      c[h][1] = a.cen[n + i] - a.cy;
      c[h][2] = a.cen[2 * n + i] - a.cz;
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) s_c[d][tid] = f2pack((float)c[0][d], (float)c[1][d]);
  }
  __syncthreads();
  const int nrows = (int)nat::min64(kTIM, a.rows - i0);
  f2r kk[NK], nkk[NK];
#pragma unroll
  for (int q = 0; q < NK; ++q) {
    kk[q] = f2pack(m.k[q], m.k[q]);
    nkk[q] = f2pack(-m.k[q], -m.k[q]);
  }
  const bool rhs = a.n_rhs > 0;
  f2r br[TP][NK], bi[TP][NK];
#pragma unroll
  for (int t = 0; t < TP; ++t)
#pragma unroll
    for (int q = 0; q < NK; ++q) br[t][q] = bi[t][q] = 0ull;
#pragma unroll 1
  for (int cc = 0; cc < kCC; ++cc) {
    const int64_t j = (int64_t)blockIdx.x * (kThreads * kCC) + cc * kThreads + tid;
    const bool valid = j < n;
    const int64_t jj = valid ? j : 0;
    f2r y[NQ][3], w[NQ], yn[NQ];
    const float nxs = a.cols.nrm[jj], nys = a.cols.nrm[n + jj], nzs = a.cols.nrm[2 * n + jj];
    const f2r nx = f2pack(nxs, nxs), ny = f2pack(nys, nys), nz = f2pack(nzs, nzs);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float v[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        v[d] = a.cols.qxyz[((size_t)q * 3 + d) * n + jj];
        y[q][d] = f2pack(v[d], v[d]);
      }
      const float wv = valid ? a.cols.qw[(size_t)q * n + jj] : 0.f;
      w[q] = f2pack(wv, wv);
      const float vn = fmaf(v[2], nzs, fmaf(v[1], nys, v[0] * nxs));
      yn[q] = f2pack(vn, vn);
    }
    f2r gr = 0ull, gi = 0ull, ngi = 0ull;
    if (rhs) {
      const double2 gv = valid ? a.g[jj] : make_double2(0.0, 0.0);
      gr = f2pack((float)gv.x, (float)gv.x);
      gi = f2pack((float)gv.y, (float)gv.y);
      ngi = f2pack(-(float)gv.y, -(float)gv.y);
    }
#pragma unroll
    for (int t = 0; t < TP; ++t) {
      if (2 * t >= nrows) continue;
      const f2r cx = s_c[0][t], cy = s_c[1][t], cz = s_c[2][t];
      const f2r cn = f2fma(cz, nz, f2fma(cy, ny, f2mul(cx, nx)));
      f2r Vr[NK], Vi[NK], Kr[NK], Ki[NK];  // K here is -K
#pragma unroll
      for (int q = 0; q < NK; ++q) Vr[q] = Vi[q] = Kr[q] = Ki[q] = 0ull;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const f2r dx = f2sub(y[q][0], cx), dy = f2sub(y[q][1], cy), dz = f2sub(y[q][2], cz);
        const f2r r2 = f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx)));
        const f2r dn = f2sub(yn[q], cn);
        const f2r rho = f2pack(nat::pair_rsqrt(f2lo(r2)), nat::pair_rsqrt(f2hi(r2)));
        const f2r rr = f2mul(r2, rho);
        const f2r tw = f2mul(w[q], rho);
        const f2r u = f2mul(tw, f2mul(dn, f2mul(rho, rho)));
#pragma unroll
        for (int kw = 0; kw < NK; ++kw) {
          const f2r kr = f2mul(rr, kk[kw]), nkr = f2mul(rr, nkk[kw]);
          float s0, c0, s1, c1;
          __sincosf(f2lo(kr), &s0, &c0);
          __sincosf(f2hi(kr), &s1, &c1);
          const f2r sn = f2pack(s0, s1), cs = f2pack(c0, c1);
          Vr[kw] = f2fma(tw, cs, Vr[kw]);
          Vi[kw] = f2fma(tw, sn, Vi[kw]);
          Kr[kw] = f2fma(u, f2fma(kr, sn, cs), Kr[kw]);
          Ki[kw] = f2fma(u, f2fma(nkr, cs, sn), Ki[kw]);
        }
      }
      const int64_t ri = a.row_begin + i0 + 2 * t;
      const bool z0 = !valid || (kCentroidRule<NQ> && j == ri), z1 = !valid || (kCentroidRule<NQ> && j == ri + 1);
#pragma unroll
      for (int kw = 0; kw < NK; ++kw) {
        if (z0 || z1) {  // padding columns (and the centroid rules' self pair) -> 0, NaN-safe
          Vr[kw] = f2pack(z0 ? 0.f : f2lo(Vr[kw]), z1 ? 0.f : f2hi(Vr[kw]));
          Vi[kw] = f2pack(z0 ? 0.f : f2lo(Vi[kw]), z1 ? 0.f : f2hi(Vi[kw]));
          Kr[kw] = f2pack(z0 ? 0.f : f2lo(Kr[kw]), z1 ? 0.f : f2hi(Kr[kw]));
          Ki[kw] = f2pack(z0 ? 0.f : f2lo(Ki[kw]), z1 ? 0.f : f2hi(Ki[kw]));
        }
        if (valid) {
          float2* arow = m.A[kw] + (size_t)(i0 + 2 * t) * a.lda + j;
          arow[0] = make_float2(f2lo(Kr[kw]), f2lo(Ki[kw]));
          if (2 * t + 1 < nrows) arow[a.lda] = make_float2(f2hi(Kr[kw]), f2hi(Ki[kw]));
        }
        br[t][kw] = f2fma(Vr[kw], gr, f2fma(Vi[kw], ngi, br[t][kw]));
        bi[t][kw] = f2fma(Vr[kw], gi, f2fma(Vi[kw], gr, bi[t][kw]));
      }
    }
  }
  if (!rhs) return;
#pragma unroll
  for (int t = 0; t < kTIM; ++t)
#pragma unroll
    for (int kw = 0; kw < NK; ++kw) {
      const f2r pr = br[t / 2][kw], pi = bi[t / 2][kw];
      double vx = (double)((t & 1) ? f2hi(pr) : f2lo(pr)), vy = (double)((t & 1) ? f2hi(pi) : f2lo(pi));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        vx += __shfl_xor_sync(0xffffffffu, vx, o);
        vy += __shfl_xor_sync(0xffffffffu, vy, o);
      }
      if (lane == 0) s_red[warp][t][kw] = make_double2(vx, vy);
    }
  __syncthreads();
  if (tid < kTIM * NK) {
    const int t = tid / NK, kw = tid % NK;
    if (t < nrows) {
      double2 sum = s_red[0][t][kw];
      for (int wv = 1; wv < kThreads / 32; ++wv) {
        sum.x += s_red[wv][t][kw].x;
        sum.y += s_red[wv][t][kw].y;
      }
      m.bpart[kw][(size_t)blockIdx.x * a.rows + i0 + t] = make_double2(-sum.x, -sum.y);  // b = -V g
    }
  }
}

template <typename R, int NQ, int NR>
void launch_far(dim3 grid, const FarArgs<R>& fa, bool bm, bool gal, cudaStream_t s) {
  if (bm) {
    far_kernel<R, NQ, NR, true><<<grid, kThreads, 0, s>>>(fa);
  } else if constexpr (sizeof(R) == 4) {
    if (gal)
      far_kernel_x2<NQ, NR, false, NQ><<<grid, kThreads, 0, s>>>(fa);
    else
      far_kernel_x2<NQ, NR><<<grid, kThreads, 0, s>>>(fa);
  } else {
    grid.y = (unsigned)((fa.rows + kTI64 - 1) / kTI64);
    if (gal)
      far_kernel<R, NQ, NR, false, false, kTI64, NQ><<<grid, kThreads, 0, s>>>(fa);
    else
      far_kernel<R, NQ, NR, false, false, kTI64><<<grid, kThreads, 0, s>>>(fa);
  }
}

template <typename R>
struct NearArgs {
  int64_t n, nv, row_begin, rows, lda, nnz;
  const int64_t* row_ptr;
  const int32_t* col;
  const uint8_t* cls;
  const double* vx;
  const int32_t* tri;
  const double* cen;
  const double* nrm;
  const double* area;
  const double4* rule;     // near rule points (parent barycentrics, weight)
  const float4* rule_f;    // the same rule in fp32 (fp32 path)
  int npts;
  const int2* items;       // compacted (entry, row) list of this launch's class
  const int32_t* nitems;   // [device] its length
  FarCols<R> cols;         // far rule (to subtract the far contribution from b)
  double cx, cy, cz;
  R k;
  int n_rhs;
  const double2* g;
  void* A;
  double2* corr;           // [nnz][n_rhs]
  double2* delta;          // matrix-free (NEXT-3): [nnz] A^near_ij - A^far_ij instead of storing A
};

// One G-lane group per near pair of one class (compacted list `items` = (entry, row)):
// G = 1 for class N (28 points per thread), G = 4 for class S (448 points over 4 lanes).
// The rule table is staged in shared memory (all groups walk it in the same order).
constexpr int kMaxNearPts = 7 << 8;  // up to 4 subdivision levels x 7 points (S: 448 at 3)

template <typename R, int NQ, int G, bool BM, bool MFD>
__device__ __forceinline__ void near_item(const NearArgs<R>& a, int64_t gid, int lig, const float4* s_rf,
                                          const double4* s_rd);

template <typename R, int NQ, int G, bool BM = false, bool MFD = false>
__global__ void __launch_bounds__(kThreads) near_kernel(NearArgs<R> a) {
  extern __shared__ __align__(16) unsigned char near_smem[];
  float4* s_rf = reinterpret_cast<float4*>(near_smem);
  double4* s_rd = reinterpret_cast<double4*>(near_smem);
  const int64_t nitems = *a.nitems;
  if ((int64_t)blockIdx.x * (blockDim.x / G) >= nitems) return;  // grid sized for the worst case
  for (int q = threadIdx.x; q < a.npts; q += blockDim.x) {
    if constexpr (sizeof(R) == 4)
      s_rf[q] = a.rule_f[q];
    else
      s_rd[q] = a.rule[q];
  }
  __syncthreads();
  // grid-stride over the pair groups; the item count is read on the device (no host sync)
  const int lig = threadIdx.x % G;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  for (int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G; gid < nitems; gid += stride)
    near_item<R, NQ, G, BM, MFD>(a, gid, lig, s_rf, s_rd);
}

// MFD: matrix-free corrections (a.delta) instead of storing A (compile-time, so the
// stored-matrix kernels keep their register budget)
template <typename R, int NQ, int G, bool BM, bool MFD>
__device__ __forceinline__ void near_item(const NearArgs<R>& a, int64_t gid, int lig, const float4* s_rf,
                                          const double4* s_rd) {
  const int2 item = a.items[gid];
  const int64_t e = item.x;
  const int64_t r = item.y;
  const int64_t i = a.row_begin + r;
  const int64_t j = a.col[e];
  const int64_t n = a.n;
  const double ci[3] = {a.cen[i], a.cen[n + i], a.cen[2 * n + i]};
  const int vid[3] = {a.tri[j], a.tri[n + j], a.tri[2 * n + j]};
  double v[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int d = 0; d < 3; ++d) v[p][d] = a.vx[d * a.nv + vid[p]];
  const R nx = (R)a.nrm[j], ny = (R)a.nrm[n + j], nz = (R)a.nrm[2 * n + j];
  const double wA = a.area[j] * nat::kInv4Pi;
  // Burton-Miller: the row's normal n_x (reading R-bm)
  const R mx = BM ? (R)a.nrm[i] : R(0), my = BM ? (R)a.nrm[n + i] : R(0), mz = BM ? (R)a.nrm[2 * n + i] : R(0);
  C2<R> V{R(0), R(0)}, K{R(0), R(0)}, Kp{R(0), R(0)}, W{R(0), R(0)};
  auto acc = [&](R dx, R dy, R dz, R wq) {
    if constexpr (BM)
      nat::pair_accumulate_bm<R>(dx, dy, dz, nx, ny, nz, mx, my, mz, wq, a.k, V, K, Kp, W);
    else
      nat::pair_accumulate<R>(dx, dy, dz, nx, ny, nz, wq, a.k, V.x, V.y, K.x, K.y);
  };
  if constexpr (sizeof(R) == 4) {
    // fp32 path: vertex offsets from the collocation point are formed in fp64 once per
    // pair and rounded (|v - c_i| ~ element size, so the rounding is relative to r);
    // each quadrature point is then d = l1 e1 + l2 e2 + l3 e3 in fp32
    float e[3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int c = 0; c < 3; ++c) e[p][c] = (float)(v[p][c] - ci[c]);
    const float wAf = (float)wA;
    for (int q = lig; q < a.npts; q += G) {
      const float4 L = s_rf[q];
      float d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = fmaf(L.z, e[2][c], fmaf(L.y, e[1][c], L.x * e[0][c]));
      acc(d[0], d[1], d[2], L.w * wAf);
    }
  } else {
    for (int q = lig; q < a.npts; q += G) {
      const double4 L = s_rd[q];
      R d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = (R)(((L.x * v[0][c] + L.y * v[1][c]) + L.z * v[2][c]) - ci[c]);
      acc(d[0], d[1], d[2], (R)(L.w * wA));
    }
  }
  if constexpr (G > 1) {
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
    auto red = [&](R& x) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o, G);
    };
    red(V.x);
    red(V.y);
    red(K.x);
    red(K.y);
    if constexpr (BM) {
      red(Kp.x);
      red(Kp.y);
      red(W.x);
      red(W.y);
    }
    if (lig != 0) return;
  }
  R Vr = V.x, Vi = V.y, Kr = K.x, Ki = K.y;
  if constexpr (BM) {  // A = -K - (i/k) W;  RHS operator V + (i/k) K'
    Kr = K.x - W.y / a.k;
    Ki = K.y + W.x / a.k;
    Vr = V.x - Kp.y / a.k;
    Vi = V.y + Kp.x / a.k;
  }
  if (!MFD) store_entry<R>(a.A, (size_t)r * a.lda + j, -Kr, -Ki);
  if (a.n_rhs > 0 || MFD) {
    R y[NQ][3], w[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      y[q][0] = a.cols.qxyz[((size_t)q * 3 + 0) * n + j];
      y[q][1] = a.cols.qxyz[((size_t)q * 3 + 1) * n + j];
      y[q][2] = a.cols.qxyz[((size_t)q * 3 + 2) * n + j];
      w[q] = a.cols.qw[(size_t)q * n + j];
    }
    R fVr, fVi, fKr, fKi;
    if constexpr (BM)
      far_entry_bm_rhs<R, NQ>(y, w, a.cols.nrm[j], a.cols.nrm[n + j], a.cols.nrm[2 * n + j], mx, my, mz,
                              (R)(ci[0] - a.cx), (R)(ci[1] - a.cy), (R)(ci[2] - a.cz), a.k, fVr, fVi);
    else
      far_entry<R, NQ>(y, w, a.cols.nrm[j], a.cols.nrm[n + j], a.cols.nrm[2 * n + j],
                       (R)(ci[0] - a.cx), (R)(ci[1] - a.cy), (R)(ci[2] - a.cz), a.k, fVr, fVi, fKr, fKi);
    if constexpr (MFD && !BM) {  // matrix-free: A_ij = A^far_ij + delta_e with A = -K
      a.delta[e] = make_double2((double)fKr - (double)Kr, (double)fKi - (double)Ki);
    }
    const double dVr = (double)Vr - (double)fVr, dVi = (double)Vi - (double)fVi;
    for (int q = 0; q < a.n_rhs; ++q) {
      double2 gv = a.g[(size_t)q * n + j];
      a.corr[(size_t)e * a.n_rhs + q] = make_double2(-(dVr * gv.x - dVi * gv.y), -(dVr * gv.y + dVi * gv.x));
    }
  }
}

// Polar self term (reading R-self): V_ii = 1/(4 pi) sum_e h_e int E(k h_e cosh u) du.
__device__ void self_single_layer(const double (&v)[3][3], const double (&c)[3], double k,
                                  const double* glx, const double* glw, int ngl, double& Vr,
                                  double& Vi) {
  Vr = Vi = 0.0;
  for (int e = 0; e < 3; ++e) {
    const double* A = v[e];
    const double* B = v[(e + 1) % 3];
    double ab[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
    double L = sqrt(ab[0] * ab[0] + ab[1] * ab[1] + ab[2] * ab[2]);
    double u[3] = {ab[0] / L, ab[1] / L, ab[2] / L};
    double ca[3] = {c[0] - A[0], c[1] - A[1], c[2] - A[2]};
    double tproj = ca[0] * u[0] + ca[1] * u[1] + ca[2] * u[2];
    double foot[3] = {A[0] + tproj * u[0], A[1] + tproj * u[1], A[2] + tproj * u[2]};
    double hv[3] = {c[0] - foot[0], c[1] - foot[1], c[2] - foot[2]};
    double h = sqrt(hv[0] * hv[0] + hv[1] * hv[1] + hv[2] * hv[2]);
    double s0 = (A[0] - foot[0]) * u[0] + (A[1] - foot[1]) * u[1] + (A[2] - foot[2]) * u[2];
    double s1 = (B[0] - foot[0]) * u[0] + (B[1] - foot[1]) * u[1] + (B[2] - foot[2]) * u[2];
    double u0 = asinh(s0 / h), u1 = asinh(s1 / h);
    double half = 0.5 * (u1 - u0), mid = 0.5 * (u1 + u0);
    double er = 0, ei = 0;
    for (int g = 0; g < ngl; ++g) {
      double R = h * cosh(mid + half * glx[g]);
      double x = k * R, re = 1.0, im = 0.0;
      if (x != 0.0) {
        double sx, cx, sh, ch;
        sincos(x, &sx, &cx);
        sincos(0.5 * x, &sh, &ch);
        re = sx / x;
        im = 2.0 * sh * sh / x;
      }
      er += glw[g] * re;
      ei += glw[g] * im;
    }
    Vr += h * half * er;
    Vi += h * half * ei;
  }
  Vr *= nat::kInv4Pi;
  Vi *= nat::kInv4Pi;
}

// Polar finite part of the hypersingular self term (reading R-bm-self):
// W_ii = ik/2 - 1/(4 pi) sum_e (1/h_e) int e^{ik h_e cosh u} / cosh^2 u du.
__device__ void self_hypersingular(const double (&v)[3][3], const double (&c)[3], double k, const double* glx,
                                   const double* glw, int ngl, double& Wr, double& Wi) {
  double tr = 0, ti = 0;
  for (int e = 0; e < 3; ++e) {
    const double* A = v[e];
    const double* B = v[(e + 1) % 3];
    double ab[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
    double L = sqrt(ab[0] * ab[0] + ab[1] * ab[1] + ab[2] * ab[2]);
    double u[3] = {ab[0] / L, ab[1] / L, ab[2] / L};
    double ca[3] = {c[0] - A[0], c[1] - A[1], c[2] - A[2]};
    double tproj = ca[0] * u[0] + ca[1] * u[1] + ca[2] * u[2];
    double foot[3] = {A[0] + tproj * u[0], A[1] + tproj * u[1], A[2] + tproj * u[2]};
    double hv[3] = {c[0] - foot[0], c[1] - foot[1], c[2] - foot[2]};
    double h = sqrt(hv[0] * hv[0] + hv[1] * hv[1] + hv[2] * hv[2]);
    double s0 = (A[0] - foot[0]) * u[0] + (A[1] - foot[1]) * u[1] + (A[2] - foot[2]) * u[2];
    double s1 = (B[0] - foot[0]) * u[0] + (B[1] - foot[1]) * u[1] + (B[2] - foot[2]) * u[2];
    double u0 = asinh(s0 / h), u1 = asinh(s1 / h);
    double half = 0.5 * (u1 - u0), mid = 0.5 * (u1 + u0);
    double er = 0, ei = 0;
    for (int g = 0; g < ngl; ++g) {
      const double ch = cosh(mid + half * glx[g]);
      double sn, cs;
      sincos(k * h * ch, &sn, &cs);
      const double wq = glw[g] / (ch * ch);
      er += wq * cs;
      ei += wq * sn;
    }
    tr += half * er / h;
    ti += half * ei / h;
  }
  Wr = -tr * nat::kInv4Pi;
  Wi = 0.5 * k - ti * nat::kInv4Pi;
}

template <typename R, int NQ, bool BM = false>
__global__ void self_kernel(int64_t n, int64_t nv, int64_t row_begin, int64_t rows, int64_t lda,
                            const double* __restrict__ vx, const int32_t* __restrict__ tri,
                            const double* __restrict__ cen, const double* __restrict__ nrm_rows,
                            FarCols<R> cols, double cx, double cy,
                            double cz, double k, const double* glx, const double* glw, int ngl,
                            int n_rhs, const double2* __restrict__ g, void* A,
                            double2* __restrict__ corr_self, double2* __restrict__ diag_delta) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int64_t i = row_begin + r;
  double v[3][3], c[3] = {cen[i], cen[n + i], cen[2 * n + i]};
  for (int p = 0; p < 3; ++p) {
    int vi = tri[p * n + i];
    for (int d = 0; d < 3; ++d) v[p][d] = vx[d * nv + vi];
  }
  if constexpr (BM) {  // A_ii = 1/2 - (i/k) W_ii  (K_ii = 0 on a flat triangle)
    double Wr, Wi;
    self_hypersingular(v, c, k, glx, glw, ngl, Wr, Wi);
    store_entry<R>(A, (size_t)r * lda + i, (R)(0.5 + Wi / k), (R)(-Wr / k));
  } else if (!diag_delta) {
    store_entry<R>(A, (size_t)r * lda + i, R(0.5), R(0));  // K_ii = 0 on a flat triangle
  }
  if (n_rhs == 0 && !diag_delta) return;
  R y[NQ][3], w[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    y[q][0] = cols.qxyz[((size_t)q * 3 + 0) * n + i];
    y[q][1] = cols.qxyz[((size_t)q * 3 + 1) * n + i];
    y[q][2] = cols.qxyz[((size_t)q * 3 + 2) * n + i];
    w[q] = cols.qw[(size_t)q * n + i];
  }
  R fVr, fVi, fKr, fKi;
  const R mx = (R)nrm_rows[i], my = (R)nrm_rows[n + i], mz = (R)nrm_rows[2 * n + i];
  if constexpr (kCentroidRule<NQ>)  // the far kernels zeroed the self pair: nothing to subtract
    fVr = fVi = fKr = fKi = R(0);
  else if constexpr (BM)
    far_entry_bm_rhs<R, NQ>(y, w, cols.nrm[i], cols.nrm[n + i], cols.nrm[2 * n + i], mx, my, mz, (R)(c[0] - cx),
                            (R)(c[1] - cy), (R)(c[2] - cz), (R)k, fVr, fVi);
  else
    far_entry<R, NQ>(y, w, cols.nrm[i], cols.nrm[n + i], cols.nrm[2 * n + i], (R)(c[0] - cx),
                     (R)(c[1] - cy), (R)(c[2] - cz), (R)k, fVr, fVi, fKr, fKi);
  if constexpr (!BM) {  // matrix-free: A_ii = 1/2 = A^far_ii + delta_i with A^far_ii = -K^far_ii
    if (diag_delta) diag_delta[r] = make_double2(0.5 + (double)fKr, (double)fKi);
  }
  if (n_rhs == 0) return;
  double Vr, Vi;
  self_single_layer(v, c, k, glx, glw, ngl, Vr, Vi);  // K'_ii = 0 too: the RHS operator is V_ii
  double dVr = Vr - (double)fVr, dVi = Vi - (double)fVi;
  for (int q = 0; q < n_rhs; ++q) {
    double2 gv = g[(size_t)q * n + i];
    double2 cs = make_double2(-(dVr * gv.x - dVi * gv.y), -(dVr * gv.y + dVi * gv.x));
    if constexpr (BM) {  // - (beta/2) g_i = -(i / 2k) g_i
      cs.x += gv.y / (2.0 * k);
      cs.y -= gv.x / (2.0 * k);
    }
    corr_self[(size_t)r * n_rhs + q] = cs;
  }
}

// ------------------------------------------------------------------------------------
// NEXT-2: Galerkin P0 near-field and self integrals (reading R-galerkin).
// One warp per element pair — the paper's "single CUDA block for each element-to-element
// integration" for adjacent or identical elements, at warp granularity:
//   class N  (no shared vertex): tensor product of the class-N rule on T_i and on T_j;
//   class S  (shared edge / vertex) and the self pair: Sauter-Schwab cube rules on the
//            reference triangle {0 <= x2 <= x1 <= 1}, chi(x) = a + x1 (b - a) + x2 (c - b),
//            shared vertices first (in T_i's order) so chi_i and chi_j agree on them.
// Points are formed relative to T_i's first (ordered) vertex from fp64 edge vectors, so
// d = y - x keeps its relative accuracy as r -> 0 in the fp32 path.  The lanes take rule
// points l, l+32, ...; fixed xor-tree reduction (deterministic).
// ------------------------------------------------------------------------------------
constexpr int kSSMaxOrder = 8;
constexpr int kSSRegions = 6 + 5 + 2;  // identical | edge | vertex

struct SSTable {  // [P][5] = (x1, x2, y1, y2, w) per case, w includes the cube Jacobians
  int off[4];     // case c occupies [off[c], off[c+1]); 0 identical, 1 edge, 2 vertex
};

// Host: the Sauter-Schwab rules (Sauter & Schwab, Boundary Element Methods, §5.2) with n
// Gauss-Legendre points per cube dimension; sum of the weights of each case = 1/4.
void ss_build(int n, std::vector<double>& out, SSTable& tab) {
  std::vector<double> gx, gw;
  gauss_legendre(n, gx, gw);
  for (int q = 0; q < n; ++q) {
    gx[q] = 0.5 * (gx[q] + 1.0);
    gw[q] *= 0.5;
  }
  out.clear();
  auto put = [&](double x1, double x2, double y1, double y2, double w) {
    out.push_back(x1);
    out.push_back(x2);
    out.push_back(y1);
    out.push_back(y2);
    out.push_back(w);
  };
  for (int c = 0; c < 3; ++c) {
    tab.off[c] = (int)(out.size() / 5);
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int d = 0; d < n; ++d)
          for (int e = 0; e < n; ++e) {
            const double xi = gx[a], e1 = gx[b], e2 = gx[d], e3 = gx[e];
            const double w4 = gw[a] * gw[b] * gw[d] * gw[e];
            if (c == 0) {  // identical panels: 6 regions, Jacobian xi^3 e1^2 e2
              const double f = w4 * xi * xi * xi * e1 * e1 * e2;
              put(xi, xi * (1 - e1 + e1 * e2), xi * (1 - e1 * e2 * e3), xi * (1 - e1), f);
              put(xi * (1 - e1 * e2 * e3), xi * (1 - e1), xi, xi * (1 - e1 + e1 * e2), f);
              put(xi, xi * e1 * (1 - e2 + e2 * e3), xi * (1 - e1 * e2), xi * e1 * (1 - e2), f);
              put(xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * (1 - e2 + e2 * e3), f);
              put(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * (1 - e2), f);
              put(xi, xi * e1 * (1 - e2), xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), f);
            } else if (c == 1) {  // common edge x2 = 0: 5 regions
              const double f1 = w4 * xi * xi * xi * e1 * e1, f = f1 * e2;
              put(xi, xi * e1 * e3, xi * (1 - e1 * e2), xi * e1 * (1 - e2), f1);
              put(xi, xi * e1, xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), f);
              put(xi * (1 - e1 * e2), xi * e1 * (1 - e2), xi, xi * e1 * e2 * e3, f);
              put(xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3), xi, xi * e1, f);
              put(xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3), xi, xi * e1 * e2, f);
            } else {  // common vertex (0, 0): 2 regions, Jacobian xi^3 e2
              const double f = w4 * xi * xi * xi * e2;
              put(xi, xi * e1, xi * e2, xi * e2 * e3, f);
              put(xi * e2, xi * e2 * e3, xi, xi * e1, f);
            }
          }
  }
  tab.off[3] = (int)(out.size() / 5);
}

template <typename R>
struct GalArgs {
  int64_t n, nv, row_begin, rows, lda;
  const int32_t* col;
  const double* vx;
  const int32_t* tri;
  const double* nrm;
  const double* area;
  const double4* rule_far;  // far rule (test and trial), NQ points
  const double4* rule_N;    // class-N rule (fp64, fp32)
  const float4* rule_Nf;
  int nN;
  const float4* ssx;        // Sauter-Schwab points (x1, x2, y1, y2) [P] in R's rounding ...
  const double4* ssx64;
  const double* ssw;        // ... and weights [P] (fp64, fp32)
  const float* ssw32;
  SSTable tab;
  const int2* items;        // (entry, row) of this launch's class (class lists)
  const int32_t* nitems;    // [device]
  bool cls_S;
  R k;
  int n_rhs;
  const double2* g;
  void* A;
  double2* corr;            // [nnz][n_rhs]
  double2* corr_self;       // [rows][n_rhs]
};

template <typename R>
__device__ __forceinline__ void warp_sum4(R& a, R& b, R& c, R& d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
    d += __shfl_xor_sync(0xffffffffu, d, o);
  }
}

// Integrals over T_i x T_j of (G, dG/dn_y) for one pair, warp-cooperative.  oi / oj: vertex
// indices in Sauter-Schwab order; ss_case < 0 -> tensor rule (class N).  Returns (in
// double, every lane) V, K (4 pi G form, unscaled rule sums) and the far-rule V.
// Class N: the warp stages 32 test points at a time in shared memory (broadcast reads),
// lane l owns trial point b = l (+32 ...), so the inner loop is LDS + 3 FADD + the pair.
template <typename R, int NQ>
__device__ void gal_pair(const GalArgs<R>& a, const int (&oi)[3], const int (&oj)[3], int64_t j, int ss_case,
                         double& Vr, double& Vi, double& Kr, double& Ki, double& fVr, double& fVi) {
  __shared__ __align__(16) R s_pts[8][32][4];  // per warp: test points (x, y, z, w)
  const int lane = threadIdx.x & 31, wib = (threadIdx.x >> 5) & 7;
  double P[3][3], Q[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      P[p][d] = a.vx[d * a.nv + oi[p]];
      Q[p][d] = a.vx[d * a.nv + oj[p]];
    }
  const R nx = (R)a.nrm[j], ny = (R)a.nrm[a.n + j], nz = (R)a.nrm[2 * a.n + j];
  // offsets relative to P0 in fp64, rounded once
  R pe[2][3], qe[3][3];  // pe: P1 - P0, P2 - P1 (SS) ; qe: Q0 - P0, Q1 - Q0, Q2 - Q1 (SS)
  R pv[3][3], qv[3][3];  // tensor rule: vertices minus P0
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    pe[0][d] = (R)(P[1][d] - P[0][d]);
    pe[1][d] = (R)(P[2][d] - P[1][d]);
    qe[0][d] = (R)(Q[0][d] - P[0][d]);
    qe[1][d] = (R)(Q[1][d] - Q[0][d]);
    qe[2][d] = (R)(Q[2][d] - Q[1][d]);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      pv[p][d] = (R)(P[p][d] - P[0][d]);
      qv[p][d] = (R)(Q[p][d] - P[0][d]);
    }
  }
  C2<R> V{R(0), R(0)}, K{R(0), R(0)}, F{R(0), R(0)};
  R dummy_r = R(0), dummy_i = R(0);
  if (ss_case >= 0) {
    const int b0 = a.tab.off[ss_case], b1 = a.tab.off[ss_case + 1];
    for (int q = b0 + lane; q < b1; q += 32) {
      R x1, x2, y1, y2;
      if constexpr (sizeof(R) == 4) {
        const float4 e = a.ssx[q];
        x1 = e.x, x2 = e.y, y1 = e.z, y2 = e.w;
      } else {
        const double4 e = a.ssx64[q];
        x1 = e.x, x2 = e.y, y1 = e.z, y2 = e.w;
      }
      R w;
      if constexpr (sizeof(R) == 4)
        w = a.ssw32[q];
      else
        w = a.ssw[q];
      R d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        d[c] = (qe[0][c] + (y1 * qe[1][c] + y2 * qe[2][c])) - (x1 * pe[0][c] + x2 * pe[1][c]);
      nat::pair_accumulate<R>(d[0], d[1], d[2], nx, ny, nz, w, a.k, V.x, V.y, K.x, K.y);
    }
  } else {
    const int nN = a.nN;
    for (int bb = 0; bb < nN; bb += 32) {
      const int b = bb + lane;
      R y[3] = {R(0), R(0), R(0)}, wb = R(0);
      if (b < nN) {
        const double4 M = a.rule_N[b];
#pragma unroll
        for (int c = 0; c < 3; ++c) y[c] = (R)((M.x * (double)qv[0][c] + M.y * (double)qv[1][c]) + M.z * (double)qv[2][c]);
        wb = (R)M.w;
      }
      for (int aa = 0; aa < nN; aa += 32) {
        __syncwarp();
        if (aa + lane < nN) {
          const double4 L = a.rule_N[aa + lane];
#pragma unroll
          for (int c = 0; c < 3; ++c) s_pts[wib][lane][c] = (R)(L.y * (double)pv[1][c] + L.z * (double)pv[2][c]);
          s_pts[wib][lane][3] = (R)L.w;
        }
        __syncwarp();
        const int na = min(32, nN - aa);
        if (b < nN)
          for (int t = 0; t < na; ++t) {
            const R x0 = s_pts[wib][t][0], x1 = s_pts[wib][t][1], x2 = s_pts[wib][t][2], wa = s_pts[wib][t][3];
            nat::pair_accumulate<R>(y[0] - x0, y[1] - x1, y[2] - x2, nx, ny, nz, wa * wb, a.k, V.x, V.y, K.x, K.y);
          }
      }
    }
  }
  // far-rule value of the same pair (the far kernel added it to the RHS): lanes < NQ^2
  if (lane < NQ * NQ) {
    const double4 L = a.rule_far[lane / NQ], M = a.rule_far[lane % NQ];
    R d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      d[c] = ((R)M.x * qv[0][c] + ((R)M.y * qv[1][c] + (R)M.z * qv[2][c])) -
             ((R)L.y * pv[1][c] + (R)L.z * pv[2][c]);
    nat::pair_accumulate<R>(d[0], d[1], d[2], nx, ny, nz, (R)(L.w * M.w), a.k, F.x, F.y, dummy_r, dummy_i);
  }
  double v0 = V.x, v1 = V.y, k0 = K.x, k1 = K.y, f0 = F.x, f1 = F.y, z0 = 0.0, z1 = 0.0;
  warp_sum4(v0, v1, k0, k1);
  warp_sum4(f0, f1, z0, z1);
  Vr = v0;
  Vi = v1;
  Kr = k0;
  Ki = k1;
  fVr = f0;
  fVi = f1;
}

// Near pairs of one class list: A_ij = -K_ij (Galerkin), b corrected by -(V - V^far) g_j.
template <typename R, int NQ>
__global__ void __launch_bounds__(256) gal_near_kernel(GalArgs<R> a) {
  const int64_t nitems = *a.nitems;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5); it < nitems; it += warps) {
    const int2 item = a.items[it];
    const int64_t e = item.x, r = item.y, i = a.row_begin + r, j = a.col[e];
    const int n = (int)a.n;
    const int ti[3] = {a.tri[i], a.tri[n + i], a.tri[2 * n + i]};
    const int tj[3] = {a.tri[j], a.tri[n + j], a.tri[2 * n + j]};
    int oi[3], oj[3], ss_case = -1;
    if (a.cls_S) {  // shared vertices first, in T_i's order
      int ns = 0, ni = 0, nj = 0;
      int si[3], ri[3], rj[3];
      for (int p = 0; p < 3; ++p) {
        const bool sh = ti[p] == tj[0] || ti[p] == tj[1] || ti[p] == tj[2];
        if (sh) si[ns++] = ti[p];
        else ri[ni++] = ti[p];
      }
      for (int p = 0; p < 3; ++p) {
        const bool sh = tj[p] == ti[0] || tj[p] == ti[1] || tj[p] == ti[2];
        if (!sh) rj[nj++] = tj[p];
      }
      for (int p = 0; p < ns; ++p) oi[p] = oj[p] = si[p];
      for (int p = 0; p < ni; ++p) oi[ns + p] = ri[p];
      for (int p = 0; p < nj; ++p) oj[ns + p] = rj[p];
      ss_case = ns == 2 ? 1 : 2;
    } else {
      for (int p = 0; p < 3; ++p) {
        oi[p] = ti[p];
        oj[p] = tj[p];
      }
    }
    double Vr, Vi, Kr, Ki, fVr, fVi;
    gal_pair<R, NQ>(a, oi, oj, j, ss_case, Vr, Vi, Kr, Ki, fVr, fVi);
    if ((threadIdx.x & 31) != 0) continue;
    const double Ai = a.area[i], Aj = a.area[j];
    const double sc = ss_case >= 0 ? 4.0 * Ai * Aj : Ai * Aj;  // SS: |det chi_i| |det chi_j|
    const double s4 = sc * nat::kInv4Pi;
    store_entry<R>(a.A, (size_t)r * a.lda + j, (R)(-Kr * s4), (R)(-Ki * s4));
    const double dVr = (Vr - fVr * (Ai * Aj / sc)) * s4, dVi = (Vi - fVi * (Ai * Aj / sc)) * s4;
    for (int q = 0; q < a.n_rhs; ++q) {
      const double2 gv = a.g[(size_t)q * n + j];
      a.corr[(size_t)e * a.n_rhs + q] = make_double2(-(dVr * gv.x - dVi * gv.y), -(dVr * gv.y + dVi * gv.x));
    }
  }
}

// Class-N pairs (tensor rule, no shared vertex) with kGN lanes per pair, so a warp keeps
// 32 / kGN pairs in flight (the index -> vertex load chain of one pair is longer than its
// 784 evaluations spread over a whole warp): lane l of a group owns trial points
// b = l, l + kGN, ... (up to kNB in registers per pass) and sweeps every test point.
constexpr int kGN = 4;
constexpr int kNB = 8;
template <typename R, int NQ>
__global__ void __launch_bounds__(256) gal_near_n_kernel(GalArgs<R> a) {
  const int64_t nitems = *a.nitems;
  const int lane = threadIdx.x & 31, lg = lane % kGN;
  const unsigned gmask = ((1u << kGN) - 1u) << (lane / kGN * kGN);
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / kGN);
  const int nN = a.nN;
  for (int64_t it = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kGN; it < nitems; it += groups) {
    const int2 item = a.items[it];
    const int64_t e = item.x, r = item.y, i = a.row_begin + r, j = a.col[e];
    const int n = (int)a.n;
    double P[3][3], Q[3][3];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const int vi = a.tri[p * n + i], vj = a.tri[p * n + j];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        P[p][d] = a.vx[d * a.nv + vi];
        Q[p][d] = a.vx[d * a.nv + vj];
      }
    }
    const R nx = (R)a.nrm[j], ny = (R)a.nrm[n + j], nz = (R)a.nrm[2 * n + j];
    R pv[3][3], qv[3][3];  // vertices minus P0, rounded once
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        pv[p][d] = (R)(P[p][d] - P[0][d]);
        qv[p][d] = (R)(Q[p][d] - P[0][d]);
      }
    C2<R> V{R(0), R(0)}, K{R(0), R(0)}, F{R(0), R(0)};
    R dr = R(0), di = R(0);
    for (int b0 = lg; b0 < nN; b0 += kGN * kNB) {
      R y[kNB][3], wb[kNB];
#pragma unroll
      for (int u = 0; u < kNB; ++u) {
        const int b = b0 + u * kGN;
        if (b < nN) {
          R Mx, My, Mz, Mw;
          if constexpr (sizeof(R) == 4) {
            const float4 M = a.rule_Nf[b];
            Mx = M.x, My = M.y, Mz = M.z, Mw = M.w;
          } else {
            const double4 M = a.rule_N[b];
            Mx = M.x, My = M.y, Mz = M.z, Mw = M.w;
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) y[u][c] = Mx * qv[0][c] + (My * qv[1][c] + Mz * qv[2][c]);
          wb[u] = Mw;
        } else {
          y[u][0] = y[u][1] = y[u][2] = R(1e3);  // far away, zero weight
          wb[u] = R(0);
        }
      }
      for (int t = 0; t < nN; ++t) {
        R Lx, Ly, Lz, Lw;
        if constexpr (sizeof(R) == 4) {
          const float4 L = a.rule_Nf[t];
          Ly = L.y, Lz = L.z, Lw = L.w;
          (void)Lx;
        } else {
          const double4 L = a.rule_N[t];
          Ly = L.y, Lz = L.z, Lw = L.w;
          (void)Lx;
        }
        R x[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) x[c] = Ly * pv[1][c] + Lz * pv[2][c];
#pragma unroll
        for (int u = 0; u < kNB; ++u)
          nat::pair_accumulate<R>(y[u][0] - x[0], y[u][1] - x[1], y[u][2] - x[2], nx, ny, nz, Lw * wb[u], a.k, V.x,
                                  V.y, K.x, K.y);
      }
    }
    for (int q = lg; q < NQ * NQ; q += kGN) {  // far-rule value of the pair
      const double4 L = a.rule_far[q / NQ], M = a.rule_far[q % NQ];
      R d[3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
        d[c] = ((R)M.x * qv[0][c] + ((R)M.y * qv[1][c] + (R)M.z * qv[2][c])) -
               ((R)L.y * pv[1][c] + (R)L.z * pv[2][c]);
      nat::pair_accumulate<R>(d[0], d[1], d[2], nx, ny, nz, (R)(L.w * M.w), a.k, F.x, F.y, dr, di);
    }
    double v[6] = {V.x, V.y, K.x, K.y, F.x, F.y};
#pragma unroll
    for (int o = kGN / 2; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 6; ++q) v[q] += __shfl_xor_sync(gmask, v[q], o, kGN);
    if (lg != 0) continue;
    const double Ai = a.area[i], Aj = a.area[j];
    const double s4 = Ai * Aj * nat::kInv4Pi;
    store_entry<R>(a.A, (size_t)r * a.lda + j, (R)(-v[2] * s4), (R)(-v[3] * s4));
    const double dVr = (v[0] - v[4]) * s4, dVi = (v[1] - v[5]) * s4;
    for (int q = 0; q < a.n_rhs; ++q) {
      const double2 gv = a.g[(size_t)q * n + j];
      a.corr[(size_t)e * a.n_rhs + q] = make_double2(-(dVr * gv.x - dVi * gv.y), -(dVr * gv.y + dVi * gv.x));
    }
  }
}

// Self pairs (Sauter-Schwab identical panels): A_ii = |T_i| / 2 (K_ii = 0, flat), b corrected
// by -V_ii g_i (the far kernel skipped the diagonal).
template <typename R, int NQ>
__global__ void __launch_bounds__(256) gal_self_kernel(GalArgs<R> a) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= a.rows) return;
  const int64_t i = a.row_begin + r;
  const int n = (int)a.n;
  const int oi[3] = {a.tri[i], a.tri[n + i], a.tri[2 * n + i]};
  double Vr, Vi, Kr, Ki, fVr, fVi;
  gal_pair<R, NQ>(a, oi, oi, i, 0, Vr, Vi, Kr, Ki, fVr, fVi);
  if ((threadIdx.x & 31) != 0) return;
  const double Ai = a.area[i];
  store_entry<R>(a.A, (size_t)r * a.lda + i, (R)(0.5 * Ai), R(0));
  const double s4 = 4.0 * Ai * Ai * nat::kInv4Pi;
  const double dVr = Vr * s4, dVi = Vi * s4;
  for (int q = 0; q < a.n_rhs; ++q) {
    const double2 gv = a.g[(size_t)q * n + i];
    a.corr_self[(size_t)r * a.n_rhs + q] = make_double2(-(dVr * gv.x - dVi * gv.y), -(dVr * gv.y + dVi * gv.x));
  }
}

// Per-class compaction of the near list (CSR order kept): cnt[c][r+1] = entries of class
// c+1 in row r; after the scan, fill writes (entry, row) pairs into the class lists.
__global__ void class_count_kernel(int64_t rows, const int64_t* __restrict__ rp, const uint8_t* __restrict__ cls,
                                   int32_t* __restrict__ cntS, int32_t* __restrict__ cntN) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int s = 0, nn = 0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
    if (cls[e] == 1) ++s;
    else ++nn;
  }
  cntS[r + 1] = s;
  cntN[r + 1] = nn;
  if (r == 0) cntS[0] = cntN[0] = 0;
}

// In-place inclusive scan of cnt[1..rows] (cnt[0] = 0); blockIdx.x selects the array
// (class S / class N counts, one launch).
__global__ void __launch_bounds__(1024) scan_i32_kernel(int32_t* cntS, int32_t* cntN, int64_t rows) {
  __shared__ int64_t sh[33];
  int32_t* cnt = blockIdx.x == 0 ? cntS : cntN;
  const int t = threadIdx.x;
  const int64_t per = (rows + 1023) / 1024;
  const int64_t b = 1 + t * per, e = nat::min64(rows + 1, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += cnt[i];
  int64_t acc = nat::block_exscan_1024(s, sh, nullptr);
  for (int64_t i = b; i < e; ++i) {
    acc += cnt[i];
    cnt[i] = (int32_t)acc;
  }
}

__global__ void class_fill_kernel(int64_t rows, const int64_t* __restrict__ rp, const uint8_t* __restrict__ cls,
                                  const int32_t* __restrict__ offS, const int32_t* __restrict__ offN,
                                  int2* __restrict__ listS, int2* __restrict__ listN) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  int s = offS[r], nn = offN[r];
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
    if (cls[e] == 1)
      listS[s++] = make_int2((int)e, (int)r);
    else
      listN[nn++] = make_int2((int)e, (int)r);
  }
}

__global__ void rhs_final_kernel(int64_t rows, int n_rhs, int n_colblk, const double2* __restrict__ bpart,
                                 const int64_t* __restrict__ rp, const double2* __restrict__ corr,
                                 const double2* __restrict__ corr_self, double2* __restrict__ b) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * n_rhs) return;
  int q = (int)(t / rows);
  int64_t r = t % rows;
  double2 s = make_double2(0.0, 0.0);
  for (int cb = 0; cb < n_colblk; ++cb) {
    double2 v = bpart[((size_t)cb * n_rhs + q) * rows + r];
    s.x += v.x;
    s.y += v.y;
  }
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
    double2 v = corr[(size_t)e * n_rhs + q];
    s.x += v.x;
    s.y += v.y;
  }
  double2 v = corr_self[(size_t)r * n_rhs + q];
  s.x += v.x;
  s.y += v.y;
  b[(size_t)q * rows + r] = s;
}

// ------------------------------------------------------------------------------------
// a6: y = A x, fp64 accumulation; CTA = 8 rows x 256 threads, x reused across rows.
// ------------------------------------------------------------------------------------
constexpr int kGemvRows = 4;   // c128 kernel: rows per cluster
constexpr int kGemvCS = 4;     // c128 kernel: column chunks = CTAs per cluster
constexpr int kGemvRows32 = 4; // c64 kernel

// c64 (NAT_FP32) matvec, HBM-bound: CTA = 4 rows x 256 threads, each thread streams two
// float4 (= 4 complex) per row per iteration with streaming loads (8 LDG.128 in flight),
// x (c128) is converted to fp32 once per column pair and reused by the 4 rows; products
// are accumulated in fp32 over 8 columns and flushed into fp64 accumulators (the matrix
// itself carries fp32 rounding, so this keeps the matvec error at the c64 level while the
// register budget allows 4 CTAs/SM); fixed-order reduction -> deterministic.
__global__ void __launch_bounds__(kThreads, 3) gemv_c64_kernel(int64_t rows, int64_t n, const float2* __restrict__ A,
                                                              int64_t lda, const double2* __restrict__ x,
                                                              double2* __restrict__ y,
                                                              const unsigned long long* __restrict__ skip) {
  if (skip && *skip == 0ull) return;  // Krylov driver: every system already converged
  constexpr int RB = kGemvRows32;
  __shared__ double2 red[kThreads / 32][RB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nr = (int)nat::min64(RB, rows - r0);
  double ar[RB], ai[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) ar[r] = ai[r] = 0.0;
  const int64_t n2 = n / 2;
  const float4* A4 = reinterpret_cast<const float4*>(A);
  const int64_t lda2 = lda / 2;
  // rows past the end re-read the last valid row (results discarded)
  const float4* const A0 = A4 + (r0 + 0) * lda2;
  const float4* const A1 = A4 + (r0 + (1 < nr ? 1 : 0)) * lda2;
  const float4* const A2 = A4 + (r0 + (2 < nr ? 2 : 0)) * lda2;
  const float4* const A3 = A4 + (r0 + (3 < nr ? 3 : 0)) * lda2;
  static_assert(RB == 4, "row pointers below assume 4 rows");
#define NAT_AROW(r) ((r) == 0 ? A0 : (r) == 1 ? A1 : (r) == 2 ? A2 : A3)
  int64_t c = tid;
  float sr[RB], si[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) sr[r] = si[r] = 0.f;
  int nacc = 0;
  for (; c + kThreads < n2; c += 2 * kThreads) {
    float4 av[2][RB];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int r = 0; r < RB; ++r) av[u][r] = __ldcs(&NAT_AROW(r)[c + u * kThreads]);
    float xr[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double2 x0 = __ldg(&x[2 * (c + u * kThreads)]), x1 = __ldg(&x[2 * (c + u * kThreads) + 1]);
      xr[u][0] = (float)x0.x;
      xr[u][1] = (float)x0.y;
      xr[u][2] = (float)x1.x;
      xr[u][3] = (float)x1.y;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 a = av[u][r];
        sr[r] = fmaf(a.x, xr[u][0], fmaf(-a.y, xr[u][1], fmaf(a.z, xr[u][2], fmaf(-a.w, xr[u][3], sr[r]))));
        si[r] = fmaf(a.x, xr[u][1], fmaf(a.y, xr[u][0], fmaf(a.z, xr[u][3], fmaf(a.w, xr[u][2], si[r]))));
      }
    }
    if (++nacc == 4) {  // flush 16 complex products per row into fp64
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        ar[r] += (double)sr[r];
        ai[r] += (double)si[r];
        sr[r] = si[r] = 0.f;
      }
      nacc = 0;
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    ar[r] += (double)sr[r];
    ai[r] += (double)si[r];
  }
  for (; c < n2; c += kThreads) {
    const double2 x0 = __ldg(&x[2 * c]), x1 = __ldg(&x[2 * c + 1]);
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const float4 a = __ldcs(&NAT_AROW(r)[c]);
      ar[r] += (double)a.x * x0.x - (double)a.y * x0.y + (double)a.z * x1.x - (double)a.w * x1.y;
      ai[r] += (double)a.x * x0.y + (double)a.y * x0.x + (double)a.z * x1.y + (double)a.w * x1.x;
    }
  }
  if ((n & 1) && tid == 0) {
    const double2 xl = x[n - 1];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (r < nr) {
        float2 a = A[(r0 + r) * lda + n - 1];
        ar[r] += (double)a.x * xl.x - (double)a.y * xl.y;
        ai[r] += (double)a.x * xl.y + (double)a.y * xl.x;
      }
    }
  }
#undef NAT_AROW
#pragma unroll
  for (int r = 0; r < RB; ++r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
      ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
    }
    if (lane == 0) red[warp][r] = make_double2(ar[r], ai[r]);
  }
  __syncthreads();
  if (tid < nr) {
    double2 s = red[0][tid];
    for (int w = 1; w < kThreads / 32; ++w) {
      s.x += red[w][tid].x;
      s.y += red[w][tid].y;
    }
    y[r0 + tid] = s;
  }
}

// c128 GEMV: a cluster of kGemvCS CTAs shares one block of kGemvRows rows, each CTA one
// of kGemvCS fixed column chunks; the chunk partials are summed through distributed shared
// memory by the cluster's rank-0 CTA in chunk order.  Fixed chunking (independent of the
// number of rows) keeps every row's summation order, and so y, identical for any row
// split (bit-identical GMRES iterates across GPU counts).
__global__ void __cluster_dims__(kGemvCS, 1, 1) __launch_bounds__(kThreads)
    gemv_c128_kernel(int64_t rows, int64_t n, const double2* __restrict__ A, int64_t lda,
                     const double2* __restrict__ x, double2* __restrict__ y,
                     const unsigned long long* __restrict__ skip) {
  if (skip && *skip == 0ull) return;  // uniform over the grid: whole clusters return
  __shared__ double2 red[kThreads / 32][kGemvRows];
  __shared__ double2 part[kGemvRows];
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk = (int)cl.block_rank();
  const int64_t r0 = (int64_t)(blockIdx.x / kGemvCS) * kGemvRows;
  const int nr = (int)nat::min64(kGemvRows, rows - r0);
  const int64_t clen = (n + kGemvCS - 1) / kGemvCS;
  const int64_t c0 = chunk * clen, c1 = nat::min64(n, c0 + clen);
  // rows past the end re-read the last valid row (results discarded)
  const double2* Ar[kGemvRows];
#pragma unroll
  for (int r = 0; r < kGemvRows; ++r) Ar[r] = A + (r0 + (r < nr ? r : 0)) * lda;
  double ar[kGemvRows], ai[kGemvRows];
#pragma unroll
  for (int r = 0; r < kGemvRows; ++r) ar[r] = ai[r] = 0.0;
  int64_t c = c0 + tid;
  for (; c + kThreads < c1; c += 2 * kThreads) {  // 2 x (kGemvRows + 1) 16-byte loads in flight
    double2 av[2][kGemvRows], xv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      xv[u] = __ldg(&x[c + u * kThreads]);
#pragma unroll
      for (int r = 0; r < kGemvRows; ++r) av[u][r] = __ldcs(&Ar[r][c + u * kThreads]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int r = 0; r < kGemvRows; ++r) {
        ar[r] = fma(av[u][r].x, xv[u].x, fma(-av[u][r].y, xv[u].y, ar[r]));
        ai[r] = fma(av[u][r].x, xv[u].y, fma(av[u][r].y, xv[u].x, ai[r]));
      }
  }
  for (; c < c1; c += kThreads) {
    const double2 xv = __ldg(&x[c]);
#pragma unroll
    for (int r = 0; r < kGemvRows; ++r) {
      const double2 av = __ldcs(&Ar[r][c]);
      ar[r] = fma(av.x, xv.x, fma(-av.y, xv.y, ar[r]));
      ai[r] = fma(av.x, xv.y, fma(av.y, xv.x, ai[r]));
    }
  }
#pragma unroll
  for (int r = 0; r < kGemvRows; ++r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ar[r] += __shfl_xor_sync(0xffffffffu, ar[r], o);
      ai[r] += __shfl_xor_sync(0xffffffffu, ai[r], o);
    }
    if (lane == 0) red[warp][r] = make_double2(ar[r], ai[r]);
  }
  __syncthreads();
  if (tid < kGemvRows) {
    double2 s = red[0][tid];
    for (int w = 1; w < kThreads / 32; ++w) {
      s.x += red[w][tid].x;
      s.y += red[w][tid].y;
    }
    part[tid] = s;
  }
  cl.sync();
  if (chunk == 0 && tid < nr) {
    double2 s = part[tid];
    for (int q = 1; q < kGemvCS; ++q) {
      const double2 v = cl.map_shared_rank(part, q)[tid];
      s.x += v.x;
      s.y += v.y;
    }
    y[r0 + tid] = s;
  }
  cl.sync();  // the other CTAs' shared memory stays alive until rank 0 has read it
}

// ------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------
struct AsmWs {
  double4* rule_far;
  double4* rule_S;
  double4* rule_N;
  float4* rule_Sf;
  float4* rule_Nf;
  double* gl;     // [2][ngl]
  void* qxyz;
  void* qw;
  void* qn;
  int32_t* cntS;   // [rows+1] per-class counts -> offsets
  int32_t* cntN;
  int2* listS;     // compacted (entry, row) lists
  int2* listN;
  double2* bpart;
  double2* corr;
  double2* corr_self;
  float4* ssx;     // Galerkin: Sauter-Schwab points (x1, x2, y1, y2) fp32 / fp64, weights
  double4* ssx64;
  double* ssw;
  float* ssw32;
};

size_t carve(nat::Carver& c, AsmWs& w, int64_t n, int64_t rows, int64_t nnz, int n_rhs, int nfar,
             int nS, int nN, int ngl, size_t rsz) {
  int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
  w.rule_far = c.take<double4>(kMaxFarQ);
  w.rule_S = c.take<double4>(nS);
  w.rule_N = c.take<double4>(nN);
  w.gl = c.take<double>(2 * (size_t)ngl);
  w.rule_Sf = c.take<float4>(nS);
  w.rule_Nf = c.take<float4>(nN);
  w.qxyz = c.take<char>(rsz * kMaxFarQ * 3 * n);
  w.qw = c.take<char>(rsz * kMaxFarQ * n);
  w.qn = c.take<char>(rsz * 3 * n);
  w.cntS = c.take<int32_t>(rows + 1);
  w.cntN = c.take<int32_t>(rows + 1);
  w.listS = c.take<int2>(nnz > 0 ? nnz : 1);
  w.listN = c.take<int2>(nnz > 0 ? nnz : 1);
  w.bpart = c.take<double2>((size_t)n_colblk * (n_rhs > 0 ? n_rhs : 1) * rows);
  w.corr = c.take<double2>((size_t)(nnz > 0 ? nnz : 1) * (n_rhs > 0 ? n_rhs : 1));
  w.corr_self = c.take<double2>((size_t)rows * (n_rhs > 0 ? n_rhs : 1));
  const size_t ssn = (size_t)kSSRegions * kSSMaxOrder * kSSMaxOrder * kSSMaxOrder * kSSMaxOrder;
  w.ssx = c.take<float4>(ssn);
  w.ssx64 = c.take<double4>(ssn);
  w.ssw = c.take<double>(ssn);
  w.ssw32 = c.take<float>(ssn);
  return c.bytes();
}

// Immutable pinned host copies of rule tables, built once per option set and process:
// every call copies its tables into the workspace with an asynchronous copy from pinned
// memory (no pageable staging, no host stall).  Entries are never freed or modified.
struct PinnedBlob {
  void* ptr = nullptr;
  size_t bytes = 0;
};
const PinnedBlob* pinned_blob(const std::tuple<int, int, int, int, int, int>& key,
                              const std::vector<char>& (*build)(const std::tuple<int, int, int, int, int, int>&)) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int>, PinnedBlob> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return &it->second;
  const std::vector<char>& src = build(key);
  PinnedBlob b;
  b.bytes = src.size();
  if (cudaHostAlloc(&b.ptr, b.bytes > 0 ? b.bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::memcpy(b.ptr, src.data(), b.bytes);
  return &(cache[key] = b);
}

constexpr int kMaxLevel = 4;
constexpr int kMaxGL = 64;

// Matrix-free outputs (NEXT-3): with `delta` set, assemble_impl writes the near/self
// corrections of the operator A = A^far + (delta on the near list and the diagonal)
// instead of A (A is not touched; the far kernel only runs for the RHS).
struct MfOut {
  double2* delta = nullptr;  // [nnz]
  double2* diag = nullptr;   // [rows]
};

template <typename R, int NQ>
nat_status assemble_impl(const nat_mesh* mesh, const nat_geom* geom, const Opts& o,
                         const int64_t* rp, const int32_t* col, const uint8_t* cls, int64_t nnz, double k,
                         int64_t row_begin, int64_t rows, int n_rhs, const double2* g, void* A,
                         int64_t lda, double2* rhs, AsmWs& w, const std::vector<Pt>& pS,
                         const std::vector<Pt>& pN, cudaStream_t s, MfOut mf = MfOut{},
                         const SSTable* ss_tab = nullptr, bool far_done = false) {
  const int64_t n = mesh->n_tri;
  const double cx = geom->center[0], cy = geom->center[1], cz = geom->center[2];
  FarCols<R> cols{(const R*)w.qxyz, (const R*)w.qw, (const R*)w.qn};
  if (!far_done) {
  far_prep_kernel<R><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      mesh->n_vert, n, mesh->vxyz, mesh->tri, geom->normal, geom->area, w.rule_far, NQ, cx, cy, cz,
      (R*)w.qxyz, (R*)w.qw, (R*)w.qn);
  NAT_LAUNCH_CHECK();
  }
  // a4: far rule on every pair, RHS partial sums
  FarArgs<R> fa{};
  fa.n = n;
  fa.row_begin = row_begin;
  fa.rows = rows;
  fa.lda = lda;
  fa.cols = cols;
  fa.cen = geom->centroid;
  fa.nrm = geom->normal;
  fa.cx = cx;
  fa.cy = cy;
  fa.cz = cz;
  fa.k = (R)k;
  fa.n_rhs = n_rhs;
  fa.g = g;
  fa.A = A;
  fa.bpart = w.bpart;
  fa.vx = mesh->vxyz;
  fa.tri = mesh->tri;
  fa.nv = mesh->n_vert;
  fa.area = geom->area;
  fa.rule = w.rule_far;
  const int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
  dim3 grid((unsigned)n_colblk, (unsigned)((rows + kTI - 1) / kTI));
  const bool timed = nat::ktimer_on() && !mf.delta && !far_done;
  if (!far_done) {
  if (timed) nat::ktimer_begin(nat::kTimerFar, s);
  if (n_rhs == 0) {
    fa.store_A = true;
    if (!mf.delta) launch_far<R, NQ, 0>(grid, fa, o.bm, o.gal, s);
  } else {
    for (int q0 = 0; q0 < n_rhs; q0 += kNRmax) {
      fa.rhs0 = q0;
      fa.store_A = (q0 == 0) && !mf.delta;
      if (n_rhs - q0 >= 2)
        launch_far<R, NQ, 2>(grid, fa, o.bm, o.gal, s);
      else
        launch_far<R, NQ, 1>(grid, fa, o.bm, o.gal, s);
    }
  }
  NAT_LAUNCH_CHECK();
  if (timed)  // far rule on every pair of the row block (test points x trial points)
    nat::ktimer_end(nat::kTimerFar, s, (double)rows * (double)n * NQ * (o.gal ? NQ : 1), nullptr, 1);
  }  // far_done: the multi-wavenumber pass formed the far entries and bpart
  if (o.gal) {  // NEXT-2: Galerkin near / self integrals (warp per pair)
    GalArgs<R> ga{};
    ga.n = n;
    ga.nv = mesh->n_vert;
    ga.row_begin = row_begin;
    ga.rows = rows;
    ga.lda = lda;
    ga.col = col;
    ga.vx = mesh->vxyz;
    ga.tri = mesh->tri;
    ga.nrm = geom->normal;
    ga.area = geom->area;
    ga.rule_far = w.rule_far;
    ga.rule_N = w.rule_N;
    ga.nN = (int)pN.size();
    ga.rule_Nf = w.rule_Nf;
    ga.ssx = w.ssx;
    ga.ssx64 = w.ssx64;
    ga.ssw = w.ssw;
    ga.ssw32 = w.ssw32;
    ga.tab = *ss_tab;
    ga.k = (R)k;
    ga.n_rhs = n_rhs;
    ga.g = g;
    ga.A = A;
    ga.corr = w.corr;
    ga.corr_self = w.corr_self;
    if (nnz > 0) {
      const unsigned rb = (unsigned)((rows + 255) / 256);
      class_count_kernel<<<rb, 256, 0, s>>>(rows, rp, cls, w.cntS, w.cntN);
      scan_i32_kernel<<<2, 1024, 0, s>>>(w.cntS, w.cntN, rows);
      class_fill_kernel<<<rb, 256, 0, s>>>(rows, rp, cls, w.cntS, w.cntN, w.listS, w.listN);
      NAT_LAUNCH_CHECK();
      const unsigned gw = (unsigned)std::min<int64_t>((int64_t)nat::device_sm_count() * 16, (nnz + 7) / 8);
      ga.items = w.listS;
      ga.nitems = w.cntS + rows;
      ga.cls_S = true;
      gal_near_kernel<R, NQ><<<gw, 256, 0, s>>>(ga);
      ga.items = w.listN;
      ga.nitems = w.cntN + rows;
      ga.cls_S = false;
      const unsigned gn = (unsigned)std::min<int64_t>((int64_t)nat::device_sm_count() * 16,
                                                      (nnz + 256 / kGN - 1) / (256 / kGN));
      gal_near_n_kernel<R, NQ><<<gn, 256, 0, s>>>(ga);
      NAT_LAUNCH_CHECK();
    }
    gal_self_kernel<R, NQ><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(ga);
    NAT_LAUNCH_CHECK();
  }
  // a5: near pairs overwrite A and correct b; self term
  if (nnz > 0 && !o.gal) {
    const unsigned rb = (unsigned)((rows + 255) / 256);
    class_count_kernel<<<rb, 256, 0, s>>>(rows, rp, cls, w.cntS, w.cntN);
    scan_i32_kernel<<<2, 1024, 0, s>>>(w.cntS, w.cntN, rows);
    class_fill_kernel<<<rb, 256, 0, s>>>(rows, rp, cls, w.cntS, w.cntN, w.listS, w.listN);
    NAT_LAUNCH_CHECK();
    NearArgs<R> na{};
    na.n = n;
    na.nv = mesh->n_vert;
    na.row_begin = row_begin;
    na.rows = rows;
    na.lda = lda;
    na.nnz = nnz;
    na.row_ptr = rp;
    na.col = col;
    na.cls = cls;
    na.vx = mesh->vxyz;
    na.tri = mesh->tri;
    na.cen = geom->centroid;
    na.nrm = geom->normal;
    na.area = geom->area;
    na.cols = cols;
    na.cx = cx;
    na.cy = cy;
    na.cz = cz;
    na.k = (R)k;
    na.n_rhs = n_rhs;
    na.g = g;
    na.A = A;
    na.corr = w.corr;
    na.delta = mf.delta;
    const size_t rsz = sizeof(R) == 4 ? sizeof(float4) : sizeof(double4);
    // persistent grids (the class counts stay on the device): at most one group per item
    const int64_t cap = (int64_t)nat::device_sm_count() * 64;
    na.rule = w.rule_S;  // class S: 4 lanes per pair
    na.rule_f = w.rule_Sf;
    na.npts = (int)pS.size();
    na.items = w.listS;
    na.nitems = w.cntS + rows;
    const unsigned gS = (unsigned)std::min(cap, (nnz * 4 + kThreads - 1) / kThreads);
    if (o.bm)
      near_kernel<R, NQ, 4, true><<<gS, kThreads, na.npts * rsz, s>>>(na);
    else
      (mf.delta ? near_kernel<R, NQ, 4, false, true> : near_kernel<R, NQ, 4>)<<<gS, kThreads, na.npts * rsz, s>>>(na);
    na.rule = w.rule_N;  // class N: one thread per pair
    na.rule_f = w.rule_Nf;
    na.npts = (int)pN.size();
    na.items = w.listN;
    na.nitems = w.cntN + rows;
    const unsigned gN = (unsigned)std::min(cap, (nnz + kThreads - 1) / kThreads);
    if (o.bm)
      near_kernel<R, NQ, 1, true><<<gN, kThreads, na.npts * rsz, s>>>(na);
    else
      (mf.delta ? near_kernel<R, NQ, 1, false, true> : near_kernel<R, NQ, 1>)<<<gN, kThreads, na.npts * rsz, s>>>(na);
    NAT_LAUNCH_CHECK();
  }
  if (o.gal) {
    // done above
  } else if (o.bm)
    self_kernel<R, NQ, true><<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(
        n, mesh->n_vert, row_begin, rows, lda, mesh->vxyz, mesh->tri, geom->centroid, geom->normal, cols, cx, cy,
        cz, k, w.gl, w.gl + o.gl, o.gl, n_rhs, g, A, w.corr_self, mf.diag);
  else
    self_kernel<R, NQ><<<(unsigned)((rows + 127) / 128), 128, 0, s>>>(
        n, mesh->n_vert, row_begin, rows, lda, mesh->vxyz, mesh->tri, geom->centroid, geom->normal, cols, cx, cy,
        cz, k, w.gl, w.gl + o.gl, o.gl, n_rhs, g, A, w.corr_self, mf.diag);
  NAT_LAUNCH_CHECK();
  if (n_rhs > 0) {
    int64_t t = rows * n_rhs;
    rhs_final_kernel<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(rows, n_rhs, (int)n_colblk, w.bpart,
                                                                 rp, w.corr, w.corr_self, rhs);
    NAT_LAUNCH_CHECK();
  }
  return NAT_OK;
}

}  // namespace

extern "C" size_t nat_bem_assemble_workspace(int64_t n_tri, int64_t rows, int64_t nnz, int n_rhs) {
  nat::Carver c(nullptr);
  AsmWs w;
  int64_t nS = 7 * (1LL << (2 * kMaxLevel)), nN = nS;
  return carve(c, w, n_tri, rows, nnz, n_rhs, kMaxFarQ, (int)nS, (int)nN, kMaxGL, sizeof(double));
}

namespace {
// nat_bem_assemble and nat_bem_mf_prepare (mf.delta set: no A, corrections instead)
// Several wavenumbers in one call (nat_bem_assemble_multi): A[q], rhs + q n_rhs rows
struct MultiK {
  int n_k = 1;
  const double* k = nullptr;  // [host][n_k]
  void* const* A = nullptr;   // [host][n_k]
};

template <int NQ>
nat_status assemble_multi_fp32(const nat_mesh* mesh, const nat_geom* geom, const Opts& o, const int64_t* rp,
                               const int32_t* col, const uint8_t* cls, int64_t nnz, const MultiK& mk,
                               int64_t row_begin, int64_t rows, int n_rhs, const double2* g, int64_t lda,
                               double2* rhs, AsmWs& w, double2* extra_bpart, const std::vector<Pt>& pS,
                               const std::vector<Pt>& pN, cudaStream_t s) {
  const int64_t n = mesh->n_tri;
  const double cx = geom->center[0], cy = geom->center[1], cz = geom->center[2];
  far_prep_kernel<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      mesh->n_vert, n, mesh->vxyz, mesh->tri, geom->normal, geom->area, w.rule_far, NQ, cx, cy, cz,
      (float*)w.qxyz, (float*)w.qw, (float*)w.qn);
  NAT_LAUNCH_CHECK();
  const int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
  const size_t bp = (size_t)n_colblk * (n_rhs > 0 ? n_rhs : 1) * rows;
  FarMultiArgs m{};
  FarArgs<float>& fa = m.b;
  fa.n = n;
  fa.row_begin = row_begin;
  fa.rows = rows;
  fa.lda = lda;
  fa.cols = FarCols<float>{(const float*)w.qxyz, (const float*)w.qw, (const float*)w.qn};
  fa.cen = geom->centroid;
  fa.cx = cx;
  fa.cy = cy;
  fa.cz = cz;
  fa.n_rhs = n_rhs;
  fa.g = g;
  for (int q = 0; q < mk.n_k; ++q) {
    m.k[q] = (float)mk.k[q];
    m.A[q] = (float2*)mk.A[q];
    m.bpart[q] = q == 0 ? w.bpart : extra_bpart + (size_t)(q - 1) * bp;
  }
  const dim3 grid((unsigned)n_colblk, (unsigned)((rows + kTIM - 1) / kTIM));
  const bool timed = nat::ktimer_on();
  if (timed) nat::ktimer_begin(nat::kTimerFar, s);
  switch (mk.n_k) {
    case 2: far_kernel_multi<NQ, 2><<<grid, kThreads, 0, s>>>(m); break;
    case 3: far_kernel_multi<NQ, 3><<<grid, kThreads, 0, s>>>(m); break;
    default: far_kernel_multi<NQ, 4><<<grid, kThreads, 0, s>>>(m); break;
  }
  NAT_LAUNCH_CHECK();
  if (timed) nat::ktimer_end(nat::kTimerFar, s, (double)rows * (double)n * NQ * mk.n_k, nullptr, mk.n_k);
  // near / self corrections and the right-hand side, one wavenumber at a time
  for (int q = 0; q < mk.n_k; ++q) {
    AsmWs wq = w;
    wq.bpart = m.bpart[q];
    nat_status st = assemble_impl<float, NQ>(mesh, geom, o, rp, col, cls, nnz, mk.k[q], row_begin, rows, n_rhs, g,
                                             mk.A[q], lda, rhs ? rhs + (size_t)q * n_rhs * rows : nullptr, wq, pS,
                                             pN, s, MfOut{}, nullptr, true);
    if (st != NAT_OK) return st;
  }
  return NAT_OK;
}

nat_status assemble_entry(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                          const int64_t* near_row_ptr, const int32_t* near_col, const uint8_t* near_cls, int64_t nnz,
                          double k,
                          nat_prec prec, int64_t row_begin, int64_t row_end, int n_rhs, const void* g, void* A,
                          int64_t lda, void* rhs, void* ws, size_t ws_bytes, nat_stream_t stream, MfOut mf,
                          const MultiK* mk = nullptr) {
  NAT_REQUIRE(mesh && geom, "mesh and geom must be non-null");
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  const int64_t n = mesh->n_tri;
  NAT_REQUIRE(geom->n_tri == n && n >= 1 && n < (1LL << 31), "inconsistent n_tri");
  NAT_REQUIRE(0 <= row_begin && row_begin < row_end && row_end <= n, "bad row range");
  NAT_REQUIRE(mf.delta || lda >= n, "lda (%lld) < n_tri (%lld)", (long long)lda, (long long)n);
  NAT_REQUIRE(k >= 0.0 && k < 1e300, "k = %g must be finite and >= 0", k);
  if (mk)
    for (int q = 0; q < mk->n_k; ++q) {
      NAT_REQUIRE(mk->k[q] >= 0.0 && mk->k[q] < 1e300, "k[%d] = %g must be finite and >= 0", q, mk->k[q]);
      NAT_REQUIRE(!(opts && opts->burton_miller) || mk->k[q] > 0.0, "Burton-Miller needs k > 0 (beta = i/k)");
      NAT_REQUIRE_DEV(mk->A[q]);
    }
  NAT_REQUIRE(!(opts && opts->burton_miller) || k > 0.0, "Burton-Miller needs k > 0 (beta = i/k)");
  NAT_REQUIRE(n_rhs >= 0 && (n_rhs == 0) == (g == nullptr), "g must be NULL iff n_rhs == 0");
  Opts o = opts_of(opts);
  NAT_REQUIRE(o.far_pts == 1 || o.far_pts == 3 || o.far_pts == 6 || o.far_pts == 7,
              "far_pts must be 1, 3, 6 or 7");
  NAT_REQUIRE(o.lev_S >= 0 && o.lev_S <= kMaxLevel && o.lev_N >= 0 && o.lev_N <= kMaxLevel,
              "near levels must be in [0, %d]", kMaxLevel);
  NAT_REQUIRE(o.gl >= 2 && o.gl <= kMaxGL, "self_theta_pts must be in [2, %d]", kMaxGL);
  NAT_REQUIRE(!mf.delta || !(opts && opts->burton_miller), "the matrix-free operator is the conventional BIE only");
  NAT_REQUIRE(!(opts && opts->galerkin) || !(opts->burton_miller || mf.delta),
              "Galerkin assembly is the stored conventional BIE (no Burton-Miller / matrix-free)");
  NAT_REQUIRE(!(opts && opts->galerkin) || (opts->ss_order >= 0 && opts->ss_order <= kSSMaxOrder),
              "ss_order must be in [1, %d]", kSSMaxOrder);
  NAT_REQUIRE_DEV(near_row_ptr);
  if (mf.delta) {
    NAT_REQUIRE_DEV(mf.delta);
    NAT_REQUIRE_DEV(mf.diag);
  } else {
    NAT_REQUIRE_DEV(A);
  }
  NAT_REQUIRE_DEV(mesh->vxyz);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->centroid);
  NAT_REQUIRE_DEV(geom->normal);
  NAT_REQUIRE_DEV(geom->area);
  if (n_rhs > 0) {
    NAT_REQUIRE_DEV(g);
    NAT_REQUIRE_DEV(rhs);
  }
  const int64_t rows = row_end - row_begin;
  cudaStream_t s = (cudaStream_t)stream;
  // nnz is the caller's (nat_bem_near_count's) host value of near_row_ptr[rows]: the call
  // never reads it back (asynchronous)
  NAT_REQUIRE(nnz >= 0 && nnz < (1LL << 31), "near list has %lld entries", (long long)nnz);
  if (nnz > 0) {
    NAT_REQUIRE_DEV(near_col);
    NAT_REQUIRE_DEV(near_cls);
  }
  std::vector<Pt> pF, pS, pN;
  base_rule(o.far_pts, pF);
  composite_rule(o.lev_S, pS);
  composite_rule(o.lev_N, pN);
  std::vector<double> glx, glw;
  gauss_legendre(o.gl, glx, glw);

  nat::Carver c(ws);
  AsmWs w;
  size_t rsz = prec == NAT_FP32 ? sizeof(float) : sizeof(double);
  size_t need = carve(c, w, n, rows, nnz, n_rhs, kMaxFarQ, (int)pS.size(), (int)pN.size(), o.gl, rsz);
  double2* extra_bpart = nullptr;
  if (mk && mk->n_k > 1) {  // one more RHS partial-sum block per extra wavenumber
    const int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
    extra_bpart = c.take<double2>((size_t)(mk->n_k - 1) * n_colblk * (n_rhs > 0 ? n_rhs : 1) * rows);
    need = c.bytes();
  }
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  NAT_REQUIRE_DEV(ws);
  // rule tables -> workspace: one asynchronous copy from an immutable pinned blob built
  // once per option set (far / class-S / class-N rules, Gauss-Legendre self rule, and the
  // Sauter-Schwab points for Galerkin), laid out exactly as the workspace carve
  SSTable tab{};
  if (o.gal) {
    std::vector<double> ssv;
    ss_build(o.ss, ssv, tab);  // the case offsets (host arithmetic; the points come from the blob)
  }
  {
    char* base = reinterpret_cast<char*>(w.rule_far);
    const size_t total = (size_t)(reinterpret_cast<char*>(w.rule_Nf + pN.size()) - base);
    const auto key = std::make_tuple(o.far_pts, o.lev_S, o.lev_N, o.gl, o.gal ? o.ss : 0, 0);
    auto build = [](const std::tuple<int, int, int, int, int, int>& kk) -> const std::vector<char>& {
      static thread_local std::vector<char> blob;
      std::vector<Pt> F, S, N;
      base_rule(std::get<0>(kk), F);
      composite_rule(std::get<1>(kk), S);
      composite_rule(std::get<2>(kk), N);
      std::vector<double> glx, glw;
      gauss_legendre(std::get<3>(kk), glx, glw);
      // the same carve as assemble_entry: rule_far[kMaxFarQ] rule_S rule_N gl[2 ngl] rule_Sf rule_Nf
      nat::Carver cc(reinterpret_cast<void*>((uintptr_t)1 << 20));  // offsets only (never dereferenced)
      double4* rf = cc.take<double4>(kMaxFarQ);
      double4* rs = cc.take<double4>(S.size());
      double4* rn = cc.take<double4>(N.size());
      double* gl = cc.take<double>(2 * glx.size());
      float4* sf = cc.take<float4>(S.size());
      float4* nf = cc.take<float4>(N.size());
      const size_t tables = (size_t)(reinterpret_cast<char*>(nf + N.size()) - reinterpret_cast<char*>(rf));
      std::vector<double> ssv;
      SSTable t{};
      if (std::get<4>(kk)) ss_build(std::get<4>(kk), ssv, t);
      const size_t np = ssv.size() / 5;
      blob.assign(tables + np * (sizeof(float4) + sizeof(double4) + sizeof(double) + sizeof(float)), 0);
      auto off = [&](const void* q) { return (size_t)(reinterpret_cast<const char*>(q) - reinterpret_cast<char*>(rf)); };
      std::memcpy(blob.data() + off(rf), F.data(), F.size() * sizeof(Pt));
      std::memcpy(blob.data() + off(rs), S.data(), S.size() * sizeof(Pt));
      std::memcpy(blob.data() + off(rn), N.data(), N.size() * sizeof(Pt));
      std::vector<double> g2(glx);
      g2.insert(g2.end(), glw.begin(), glw.end());
      std::memcpy(blob.data() + off(gl), g2.data(), g2.size() * sizeof(double));
      for (size_t q = 0; q < S.size(); ++q) {
        const float4 v = make_float4((float)S[q].l1, (float)S[q].l2, (float)S[q].l3, (float)S[q].w);
        std::memcpy(blob.data() + off(sf + q), &v, sizeof v);
      }
      for (size_t q = 0; q < N.size(); ++q) {
        const float4 v = make_float4((float)N[q].l1, (float)N[q].l2, (float)N[q].l3, (float)N[q].w);
        std::memcpy(blob.data() + off(nf + q), &v, sizeof v);
      }
      // Sauter-Schwab: [np] float4 | [np] double4 | [np] double | [np] float after the tables
      char* p0 = blob.data() + tables;
      for (size_t q = 0; q < np; ++q) {
        const double* e = &ssv[5 * q];
        const float4 xf = make_float4((float)e[0], (float)e[1], (float)e[2], (float)e[3]);
        const double4 xd = make_double4(e[0], e[1], e[2], e[3]);
        const double wv = e[4];
        const float wf = (float)e[4];
        std::memcpy(p0 + q * sizeof(float4), &xf, sizeof xf);
        std::memcpy(p0 + np * sizeof(float4) + q * sizeof(double4), &xd, sizeof xd);
        std::memcpy(p0 + np * (sizeof(float4) + sizeof(double4)) + q * sizeof(double), &wv, sizeof wv);
        std::memcpy(p0 + np * (sizeof(float4) + sizeof(double4) + sizeof(double)) + q * sizeof(float), &wf, sizeof wf);
      }
      return blob;
    };
    const PinnedBlob* pb = pinned_blob(key, build);
    if (!pb) return nat::fail(NAT_ERR_CUDA, "pinned rule tables: %s", cudaGetErrorString(cudaGetLastError()));
    NAT_CUDA_TRY(cudaMemcpyAsync(base, pb->ptr, total, cudaMemcpyHostToDevice, s));
    if (o.gal) {
      const size_t np = (pb->bytes - total) / (sizeof(float4) + sizeof(double4) + sizeof(double) + sizeof(float));
      const char* p0 = reinterpret_cast<const char*>(pb->ptr) + total;
      NAT_CUDA_TRY(cudaMemcpyAsync(w.ssx, p0, np * sizeof(float4), cudaMemcpyHostToDevice, s));
      NAT_CUDA_TRY(cudaMemcpyAsync(w.ssx64, p0 + np * sizeof(float4), np * sizeof(double4), cudaMemcpyHostToDevice, s));
      NAT_CUDA_TRY(cudaMemcpyAsync(w.ssw, p0 + np * (sizeof(float4) + sizeof(double4)), np * sizeof(double),
                                   cudaMemcpyHostToDevice, s));
      NAT_CUDA_TRY(cudaMemcpyAsync(w.ssw32, p0 + np * (sizeof(float4) + sizeof(double4) + sizeof(double)),
                                   np * sizeof(float), cudaMemcpyHostToDevice, s));
    }
  }
  const double2* gg = (const double2*)g;
  double2* bb = (double2*)rhs;
  if (mk && mk->n_k > 1) {
    const bool fused = prec == NAT_FP32 && !o.bm && !o.gal && n_rhs <= 1;
    if (fused) {
#define NAT_MULTI(NQ) \
  assemble_multi_fp32<NQ>(mesh, geom, o, near_row_ptr, near_col, near_cls, nnz, *mk, row_begin, rows, n_rhs, gg, lda, \
                          bb, w, extra_bpart, pS, pN, s)
      switch (o.far_pts) {
        case 1: return NAT_MULTI(1);
        case 3: return NAT_MULTI(3);
        case 6: return NAT_MULTI(6);
        default: return NAT_MULTI(7);
      }
#undef NAT_MULTI
    }
    // other variants: one far pass per wavenumber
    for (int q = 0; q < mk->n_k; ++q) {
      nat_status st = assemble_entry(mesh, geom, opts, near_row_ptr, near_col, near_cls, nnz, mk->k[q], prec,
                                     row_begin, row_end, n_rhs, g, mk->A[q], lda,
                                     bb ? (void*)(bb + (size_t)q * n_rhs * rows) : nullptr, ws, ws_bytes, stream, mf);
      if (st != NAT_OK) return st;
    }
    return NAT_OK;
  }
#define NAT_ASM(R, NQ)                                                                         \
  assemble_impl<R, NQ>(mesh, geom, o, near_row_ptr, near_col, near_cls, nnz, k, row_begin, rows, \
                       n_rhs, gg, A, lda, bb, w, pS, pN, s, mf, &tab)
  if (prec == NAT_FP32) {
    switch (o.far_pts) {
      case 1: return NAT_ASM(float, 1);
      case 3: return NAT_ASM(float, 3);
      case 6: return NAT_ASM(float, 6);
      default: return NAT_ASM(float, 7);
    }
  } else {
    switch (o.far_pts) {
      case 1: return NAT_ASM(double, 1);
      case 3: return NAT_ASM(double, 3);
      case 6: return NAT_ASM(double, 6);
      default: return NAT_ASM(double, 7);
    }
  }
#undef NAT_ASM
}
}  // namespace

extern "C" nat_status nat_bem_assemble(const nat_mesh* mesh, const nat_geom* geom,
                                       const nat_quad_opts* opts, const int64_t* near_row_ptr,
                                       const int32_t* near_col, const uint8_t* near_cls, int64_t nnz, double k,
                                       nat_prec prec, int64_t row_begin, int64_t row_end, int n_rhs,
                                       const void* g, void* A, int64_t lda, void* rhs, void* ws,
                                       size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  return assemble_entry(mesh, geom, opts, near_row_ptr, near_col, near_cls, nnz, k, prec, row_begin, row_end, n_rhs,
                        g, A, lda, rhs, ws, ws_bytes, stream, MfOut{});
}

extern "C" size_t nat_bem_assemble_multi_workspace(int64_t n_tri, int64_t rows, int64_t nnz, int n_rhs, int n_k) {
  const size_t a = nat_bem_assemble_workspace(n_tri, rows, nnz, n_rhs);
  if (n_k <= 1) return a;
  const int64_t n_colblk = (n_tri + kThreads * kCC - 1) / (kThreads * kCC);
  return a + nat::align_up(sizeof(double2) * (size_t)(n_k - 1) * n_colblk * (n_rhs > 0 ? n_rhs : 1) * rows, 256) + 256;
}

extern "C" nat_status nat_bem_assemble_multi(const nat_mesh* mesh, const nat_geom* geom, const nat_quad_opts* opts,
                                             const int64_t* near_row_ptr, const int32_t* near_col,
                                             const uint8_t* near_cls, int64_t nnz, int n_k, const double* k,
                                             nat_prec prec, int64_t row_begin, int64_t row_end, int n_rhs,
                                             const void* g, void* const* A, int64_t lda, void* rhs, void* ws,
                                             size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(n_k >= 1 && n_k <= kMaxK && k && A, "need 1 <= n_k <= %d and host arrays k[n_k], A[n_k]", kMaxK);
  MultiK mk;
  mk.n_k = n_k;
  mk.k = k;
  mk.A = A;
  return assemble_entry(mesh, geom, opts, near_row_ptr, near_col, near_cls, nnz, k[0], prec, row_begin, row_end, n_rhs,
                        g, A[0], lda, rhs, ws, ws_bytes, stream, MfOut{}, &mk);
}

namespace {
void launch_gemv(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda, const void* x, void* y,
                 const unsigned long long* skip, cudaStream_t s) {
  if (prec == NAT_FP32) {
    const unsigned grid = (unsigned)((rows + kGemvRows32 - 1) / kGemvRows32);
    gemv_c64_kernel<<<grid, kThreads, 0, s>>>(rows, n, (const float2*)A, lda, (const double2*)x, (double2*)y, skip);
  } else {
    const unsigned grid = (unsigned)(kGemvCS * ((rows + kGemvRows - 1) / kGemvRows));
    gemv_c128_kernel<<<grid, kThreads, 0, s>>>(rows, n, (const double2*)A, lda, (const double2*)x, (double2*)y,
                                               skip);
  }
}
}  // namespace

extern "C" nat_status nat_bem_matvec(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda,
                                     const void* x, void* y, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(rows >= 1 && n >= 1 && lda >= n, "need rows, n >= 1 and lda >= n");
  NAT_REQUIRE(prec == NAT_FP64 || (lda % 2 == 0 && ((uintptr_t)A % 16) == 0),
              "NAT_FP32 matvec needs an even lda and a 16-byte aligned A");
  NAT_REQUIRE_DEV(A);
  NAT_REQUIRE_DEV(x);
  NAT_REQUIRE_DEV(y);
  launch_gemv(prec, rows, n, A, lda, x, y, nullptr, (cudaStream_t)stream);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

namespace nat {
// Used by the GMRES driver (gmres.cu).
nat_status matvec_internal(nat_prec prec, int64_t rows, int64_t n, const void* A, int64_t lda,
                           const void* x, void* y, cudaStream_t s, const unsigned long long* skip) {
  launch_gemv(prec, rows, n, A, lda, x, y, skip, s);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
}  // namespace nat

// ------------------------------------------------------------------------------------
// NEXT-3: matrix-free dense operator (include/nat.h, nat_bem_mf_*).
//   (A x)_i = sum_j A^far_ij x_j  [far kernel in MV mode, every pair, nothing stored]
//           + sum_{e in near(i)} delta_e x_col[e] + diag_i x_i   [mf_final_kernel]
// ------------------------------------------------------------------------------------
namespace {

struct MfWs {
  double4* rule_far;
  void* qxyz;
  void* qw;
  void* qn;
  double2* bpart;  // [n_colblk][rows]
};

size_t mf_carve(nat::Carver& c, MfWs& w, int64_t n, int64_t rows, size_t rsz) {
  const int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
  w.rule_far = c.take<double4>(kMaxFarQ);
  w.qxyz = c.take<char>(rsz * kMaxFarQ * 3 * n);
  w.qw = c.take<char>(rsz * kMaxFarQ * n);
  w.qn = c.take<char>(rsz * 3 * n);
  w.bpart = c.take<double2>((size_t)n_colblk * rows);
  return c.bytes();
}

// y_r = sum over column blocks of the far partial sums + the near corrections + the
// diagonal correction.  One warp per row: lane l takes column blocks l, l+32, ... and near
// entries l, l+32, ... (loads in flight together), fixed xor tree -> deterministic and
// independent of the row split.
__global__ void __launch_bounds__(256) mf_final_kernel(int64_t rows, int64_t row_begin, int n_colblk,
                                                       const double2* __restrict__ bpart,
                                                       const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                       const double2* __restrict__ delta,
                                                       const double2* __restrict__ diag,
                                                       const double2* __restrict__ x, double2* __restrict__ y,
                                                       const unsigned long long* __restrict__ skip) {
  if (skip && *skip == 0ull) return;
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;  // whole warps
  double sx = 0.0, sy = 0.0;
  for (int cb = lane; cb < n_colblk; cb += 32) {
    const double2 v = bpart[(size_t)cb * rows + r];
    sx += v.x;
    sy += v.y;
  }
  const int64_t e1 = rp[r + 1];
  for (int64_t e = rp[r] + lane; e < e1; e += 32) {
    const double2 d = delta[e], xv = x[col[e]];
    sx += d.x * xv.x - d.y * xv.y;
    sy += d.x * xv.y + d.y * xv.x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  if (lane != 0) return;
  const double2 d = diag[r], xv = x[row_begin + r];
  sx += d.x * xv.x - d.y * xv.y;
  sy += d.x * xv.y + d.y * xv.x;
  y[r] = make_double2(sx, sy);
}

nat_status mf_check(const nat_bem_mf* op) {
  NAT_REQUIRE(op && op->mesh && op->geom, "op, op->mesh and op->geom must be non-null");
  NAT_REQUIRE(op->prec == NAT_FP32 || op->prec == NAT_FP64, "bad precision %d", (int)op->prec);
  const int64_t n = op->mesh->n_tri;
  NAT_REQUIRE(op->geom->n_tri == n && n >= 1 && n < (1LL << 31), "inconsistent n_tri");
  NAT_REQUIRE(0 <= op->row_begin && op->row_begin < op->row_end && op->row_end <= n, "bad row range");
  NAT_REQUIRE(op->k >= 0.0 && op->k < 1e300, "k = %g must be finite and >= 0", op->k);
  NAT_REQUIRE(!(op->opts && op->opts->burton_miller), "the matrix-free operator is the conventional BIE only");
  const int fp = opts_of(op->opts).far_pts;
  NAT_REQUIRE(fp == 1 || fp == 3 || fp == 6 || fp == 7, "far_pts must be 1, 3, 6 or 7");
  NAT_REQUIRE_DEV(op->near_row_ptr);
  NAT_REQUIRE_DEV(op->near_delta);
  NAT_REQUIRE_DEV(op->diag_delta);
  NAT_REQUIRE_DEV(op->mesh->vxyz);
  NAT_REQUIRE_DEV(op->mesh->tri);
  NAT_REQUIRE_DEV(op->geom->centroid);
  NAT_REQUIRE_DEV(op->geom->normal);
  NAT_REQUIRE_DEV(op->geom->area);
  return NAT_OK;
}

size_t mf_ws_bytes(const nat_bem_mf* op) {
  nat::Carver c(nullptr);
  MfWs w;
  return mf_carve(c, w, op->mesh->n_tri, op->row_end - op->row_begin, op->prec == NAT_FP32 ? 4 : 8);
}

template <typename R, int NQ>
nat_status mf_launch(const nat_bem_mf* op, const MfWs& w, const double2* x, double2* y,
                     const unsigned long long* skip, cudaStream_t s) {
  const int64_t n = op->mesh->n_tri, rows = op->row_end - op->row_begin;
  FarArgs<R> fa{};
  fa.n = n;
  fa.row_begin = op->row_begin;
  fa.rows = rows;
  fa.lda = 0;
  fa.cols = FarCols<R>{(const R*)w.qxyz, (const R*)w.qw, (const R*)w.qn};
  fa.cen = op->geom->centroid;
  fa.nrm = op->geom->normal;
  fa.cx = op->geom->center[0];
  fa.cy = op->geom->center[1];
  fa.cz = op->geom->center[2];
  fa.k = (R)op->k;
  fa.n_rhs = 1;
  fa.rhs0 = 0;
  fa.g = x;
  fa.A = nullptr;
  fa.store_A = false;
  fa.bpart = w.bpart;
  fa.skip = skip;
  const int64_t n_colblk = (n + kThreads * kCC - 1) / (kThreads * kCC);
  if constexpr (sizeof(R) == 4) {
    dim3 grid((unsigned)n_colblk, (unsigned)((rows + kTI - 1) / kTI));
    far_kernel_x2<NQ, 1, true><<<grid, kThreads, 0, s>>>(fa);
  } else {
    dim3 grid((unsigned)n_colblk, (unsigned)((rows + kTI64 - 1) / kTI64));
    far_kernel<R, NQ, 1, false, true, kTI64><<<grid, kThreads, 0, s>>>(fa);
  }
  NAT_LAUNCH_CHECK();
  mf_final_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(
      rows, op->row_begin, (int)n_colblk, w.bpart, op->near_row_ptr, op->near_col, (const double2*)op->near_delta,
      (const double2*)op->diag_delta, x, y, skip);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

}  // namespace

namespace nat {
size_t mf_apply_ws(const nat_bem_mf* op) { return mf_ws_bytes(op); }

// Column rule data into the workspace (once per operator; the far points depend only on
// the mesh and the rule).
nat_status mf_begin(const nat_bem_mf* op, void* ws, size_t ws_bytes, cudaStream_t s) {
  nat_status st = mf_check(op);
  if (st != NAT_OK) return st;
  Carver c(ws);
  MfWs w;
  const int64_t n = op->mesh->n_tri;
  const size_t need = mf_carve(c, w, n, op->row_end - op->row_begin, op->prec == NAT_FP32 ? 4 : 8);
  if (ws_bytes < need) return fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  NAT_REQUIRE_DEV(ws);
  const Opts o = opts_of(op->opts);
  // the far rule from an immutable pinned blob (asynchronous copy, no pageable staging)
  auto build = [](const std::tuple<int, int, int, int, int, int>& kk) -> const std::vector<char>& {
    static thread_local std::vector<char> blob;
    std::vector<Pt> F;
    base_rule(std::get<0>(kk), F);
    blob.assign(reinterpret_cast<const char*>(F.data()), reinterpret_cast<const char*>(F.data() + F.size()));
    return blob;
  };
  const PinnedBlob* pb = pinned_blob(std::make_tuple(o.far_pts, 0, 0, 0, 0, 1), build);
  if (!pb) return fail(NAT_ERR_CUDA, "pinned rule table: %s", cudaGetErrorString(cudaGetLastError()));
  NAT_CUDA_TRY(cudaMemcpyAsync(w.rule_far, pb->ptr, pb->bytes, cudaMemcpyHostToDevice, s));
  const double cx = op->geom->center[0], cy = op->geom->center[1], cz = op->geom->center[2];
  if (op->prec == NAT_FP32)
    far_prep_kernel<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        op->mesh->n_vert, n, op->mesh->vxyz, op->mesh->tri, op->geom->normal, op->geom->area, w.rule_far, o.far_pts,
        cx, cy, cz, (float*)w.qxyz, (float*)w.qw, (float*)w.qn);
  else
    far_prep_kernel<double><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        op->mesh->n_vert, n, op->mesh->vxyz, op->mesh->tri, op->geom->normal, op->geom->area, w.rule_far, o.far_pts,
        cx, cy, cz, (double*)w.qxyz, (double*)w.qw, (double*)w.qn);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

// y[rows] = (A x) on this rank's rows; x [n] (after mf_begin on the same ws).
nat_status mf_apply(const nat_bem_mf* op, void* ws, const double2* x, double2* y, const unsigned long long* skip,
                    cudaStream_t s) {
  Carver c(ws);
  MfWs w;
  mf_carve(c, w, op->mesh->n_tri, op->row_end - op->row_begin, op->prec == NAT_FP32 ? 4 : 8);
  const int fp = opts_of(op->opts).far_pts;
#define NAT_MF(R, NQ) mf_launch<R, NQ>(op, w, x, y, skip, s)
  if (op->prec == NAT_FP32) {
    switch (fp) {
      case 1: return NAT_MF(float, 1);
      case 3: return NAT_MF(float, 3);
      case 6: return NAT_MF(float, 6);
      default: return NAT_MF(float, 7);
    }
  } else {
    switch (fp) {
      case 1: return NAT_MF(double, 1);
      case 3: return NAT_MF(double, 3);
      case 6: return NAT_MF(double, 6);
      default: return NAT_MF(double, 7);
    }
  }
#undef NAT_MF
}
}  // namespace nat

extern "C" size_t nat_bem_mf_workspace(const nat_bem_mf* op, int64_t nnz, int n_rhs) {
  if (!op || !op->mesh || op->row_end <= op->row_begin) return 0;
  const int64_t n = op->mesh->n_tri, rows = op->row_end - op->row_begin;
  const size_t a = nat_bem_assemble_workspace(n, rows, nnz, n_rhs);
  const size_t b = mf_ws_bytes(op);
  return a > b ? a : b;
}

extern "C" nat_status nat_bem_mf_prepare(const nat_bem_mf* op, int n_rhs, const void* g, void* rhs, void* ws,
                                         size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = mf_check(op);
  if (st != NAT_OK) return st;
  MfOut mf;
  mf.delta = (double2*)op->near_delta;
  mf.diag = (double2*)op->diag_delta;
  return assemble_entry(op->mesh, op->geom, op->opts, op->near_row_ptr, op->near_col, op->near_cls, op->nnz, op->k,
                        op->prec,
                        op->row_begin, op->row_end, n_rhs, g, nullptr, 0, rhs, ws, ws_bytes, stream, mf);
}

extern "C" nat_status nat_bem_mf_matvec(const nat_bem_mf* op, const void* x, void* y, void* ws, size_t ws_bytes,
                                        nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = mf_check(op);
  if (st != NAT_OK) return st;
  NAT_REQUIRE_DEV(x);
  NAT_REQUIRE_DEV(y);
  cudaStream_t s = (cudaStream_t)stream;
  st = nat::mf_begin(op, ws, ws_bytes, s);
  if (st != NAT_OK) return st;
  return nat::mf_apply(op, ws, (const double2*)x, (double2*)y, nullptr, s);
}
