// Rows a8-a10 — the Monte-Carlo BEM estimator BEM-MC (§4.1.1-4.2: Eq. BIE
// l.194-198, Eq. SYS l.200-204, the disk split and disk terms l.215-236), with the
// readings R-sign, R-mc-sample, R-eps, R-weight, R-disk of DESIGN.md §3:
//   a8  uniform-by-area samples from a Philox4x32-10 counter stream (bit-identical with
//       the oracle: every fp64 step uses round-to-nearest intrinsics, no FMA);
//   a9  b_i = -w sum_{j != i} G(y_i, y_j) g_j - (eps/2) g_i;
//   a10 (A p)_i = 1/2 p_i - w sum_{j != i} dG/dn_y(y_i, y_j) p_j   (matrix-free);
// batched over every wavenumber sharing the sample set and solved with the batched
// GMRES engine (krylov.cuh).  a9/a10 reuse the radiation kernel with targets = sources
// (TMA-staged source tiles, self pair excluded exactly).
#include <chrono>
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <future>
#include <map>
#include <mutex>
#include <queue>
#include <thread>
#include <vector>

#include "krylov.cuh"
#include "nat_internal.cuh"
#include "pair.cuh"
#include "philox.cuh"
#include "sampling.cuh"
#include "radiate.cuh"

namespace {

__global__ void mc_sample_kernel(int64_t M, uint64_t seed, uint64_t stream_id, uint32_t tag, int64_t nv, int64_t nt,
                                 const double* __restrict__ vx, const int32_t* __restrict__ tri,
                                 const double* __restrict__ nrm, const double* __restrict__ cdf,
                                 double* __restrict__ smp, int32_t* __restrict__ stri) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= M) return;
  uint32_t c0 = (uint32_t)j, c1 = tag, c2 = (uint32_t)stream_id, c3 = (uint32_t)(stream_id >> 32);
  nat::philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double two32 = 2.3283064365386963e-10;  // 2^-32
  const double u0 = __dmul_rn(__dadd_rn((double)c0, 0.5), two32);
  const double u1 = __dmul_rn(__dadd_rn((double)c1, 0.5), two32);
  const double u2 = __dmul_rn(__dadd_rn((double)c2, 0.5), two32);
  // upper_bound: first t with cdf[t] > u0 * cdf[N-1]
  const double v = __dmul_rn(u0, cdf[nt - 1]);
  int64_t lo = 0, hi = nt;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > v)
      hi = mid;
    else
      lo = mid + 1;
  }
  const int64_t t = lo < nt ? lo : nt - 1;
  const double s = __dsqrt_rn(u1);
  const double b1 = __dsub_rn(1.0, s);
  const double b2 = __dmul_rn(s, __dsub_rn(1.0, u2));
  const double b3 = __dmul_rn(s, u2);
  const int a = tri[t], b = tri[nt + t], c = tri[2 * nt + t];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double* X = vx + d * nv;
    smp[d * M + j] = __dadd_rn(__dadd_rn(__dmul_rn(b1, X[a]), __dmul_rn(b2, X[b])), __dmul_rn(b3, X[c]));
    smp[(3 + d) * M + j] = nrm[d * nt + t];
  }
  stri[j] = (int32_t)t;
}

constexpr int kCT = 256;

// Smallest (i, j), i != j, with |y_i - y_j| < 1e-12 (packed i << 32 | j), brute force.
__global__ void __launch_bounds__(kCT) coincident_kernel(int64_t M, const double* __restrict__ smp,
                                                       unsigned long long* best) {
  __shared__ double sx[kCT], sy[kCT], sz[kCT];
  const int64_t i = blockIdx.x * (int64_t)kCT + threadIdx.x;
  double xi = 0, yi = 0, zi = 0;
  if (i < M) {
    xi = smp[i];
    yi = smp[M + i];
    zi = smp[2 * M + i];
  }
  unsigned long long mine = ~0ull;
  for (int64_t j0 = 0; j0 < M; j0 += kCT) {
    __syncthreads();
    const int64_t jl = j0 + threadIdx.x;
    if (jl < M) {
      sx[threadIdx.x] = smp[jl];
      sy[threadIdx.x] = smp[M + jl];
      sz[threadIdx.x] = smp[2 * M + jl];
    }
    __syncthreads();
    const int jn = (int)nat::min64(kCT, M - j0);
    if (i < M && mine == ~0ull) {
      for (int t = 0; t < jn; ++t) {
        const double dx = xi - sx[t], dy = yi - sy[t], dz = zi - sz[t];
        if (dx * dx + dy * dy + dz * dz < 1e-24 && j0 + t != i) {
          mine = ((unsigned long long)i << 32) | (unsigned long long)(j0 + t);
          break;
        }
      }
    }
  }
  if (mine != ~0ull) atomicMin(best, mine);
}

__global__ void init_best_kernel(unsigned long long* best) { *best = ~0ull; }

__global__ void gather_g_kernel(int nsys, int64_t M, int64_t nt, const double2* __restrict__ g_tri,
                                const int32_t* __restrict__ stri, double2* __restrict__ gs) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (j >= M || s >= nsys) return;
  gs[(size_t)s * M + j] = g_tri[(size_t)s * nt + stri[j]];
}

// ---- close sample pairs (fp32 r^2 <= (2 eps)^2): evaluated in fp64 -------------------
// With random samples some pairs are far closer than the sample spacing; their fp32
// coordinates (rounded to ~6e-8 |y|) would give O(1e-3) errors in d.n and 1/r.  The fp32
// kernel skips exactly these pairs (same pair_r2_f32 on the same staged coordinates) and
// this fp64 pass adds them, so the fp32 path keeps the 1e-4 parity bar.
constexpr int kNT = 256;

// One warp per 4 rows (32 rows per CTA), candidates staged 256 at a time in shared
// memory, hits compacted with __ballot_sync (columns ascending, deterministic).
constexpr int kNW = 8, kNRows = 4;
template <bool kFill>
__global__ void __launch_bounds__(kNT) mc_near_kernel(int64_t M, const double* __restrict__ smp, double cx,
                                                      double cy, double cz, float thr,
                                                      int32_t* __restrict__ rp, int32_t* __restrict__ col,
                                                      int64_t cap, int* overflow) {
  __shared__ float sx[kNT], sy[kNT], sz[kNT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * (kNW * kNRows) + warp * kNRows;
  float xi[kNRows], yi[kNRows], zi[kNRows];
  int64_t pos[kNRows];
  bool live[kNRows];
#pragma unroll
  for (int q = 0; q < kNRows; ++q) {
    const int64_t i = r0 + q;
    live[q] = i < M;
    const int64_t ii = live[q] ? i : 0;
    xi[q] = (float)(smp[ii] - cx);
    yi[q] = (float)(smp[M + ii] - cy);
    zi[q] = (float)(smp[2 * M + ii] - cz);
    pos[q] = (kFill && live[q]) ? rp[i] : 0;
  }
  for (int64_t j0 = 0; j0 < M; j0 += kNT) {
    __syncthreads();
    const int64_t jl = j0 + threadIdx.x;
    if (jl < M) {
      sx[threadIdx.x] = (float)(smp[jl] - cx);
      sy[threadIdx.x] = (float)(smp[M + jl] - cy);
      sz[threadIdx.x] = (float)(smp[2 * M + jl] - cz);
    }
    __syncthreads();
    const int jn = (int)nat::min64(kNT, M - j0);
    for (int jj = 0; jj < jn; jj += 32) {
      const int t = jj + lane;
      const bool in = t < jn;
      const float ox = in ? sx[t] : 3e30f, oy = in ? sy[t] : 3e30f, oz = in ? sz[t] : 3e30f;
#pragma unroll
      for (int q = 0; q < kNRows; ++q) {
        if (!live[q]) continue;  // warp-uniform
        const float r2 = nat::pair_r2_f32(__fsub_rn(ox, xi[q]), __fsub_rn(oy, yi[q]), __fsub_rn(oz, zi[q]));
        const bool hit = in && r2 <= thr && j0 + t != r0 + q;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (kFill && hit) {
          const int64_t o = pos[q] + __popc(m & ((1u << lane) - 1u));
          if (o < cap) col[o] = (int32_t)(j0 + t);
        }
        pos[q] += __popc(m);
      }
    }
  }
  if (!kFill && lane == 0) {
#pragma unroll
    for (int q = 0; q < kNRows; ++q)
      if (live[q]) rp[r0 + q + 1] = (int32_t)pos[q];
  }
}

__global__ void __launch_bounds__(1024) scan32_kernel(int32_t* rp, int64_t M, int64_t cap, int* overflow) {
  __shared__ int64_t sh[33];
  const int t = threadIdx.x;
  const int64_t per = (M + 1023) / 1024;
  const int64_t b = 1 + t * per, e = nat::min64(M + 1, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += rp[i];
  int64_t total = 0;
  int64_t acc = nat::block_exscan_1024(s, sh, &total);
  if (t == 0 && total > cap) *overflow = 1;
  for (int64_t i = b; i < e; ++i) {
    acc += rp[i];
    rp[i] = (int32_t)(acc < cap ? acc : cap);
  }
  if (t == 0) rp[0] = 0;
}

// R[s][i] += w [p_s(y_j) dG_s/dn_y(y_i, y_j) - g_s(y_j) G_s(y_i, y_j)] over the close pairs
// of row i, in CSR order, fp64.
struct KArr {
  double k[64];
};

// Fused epilogue of the MC operators: sum of the split-K partials, the fp64 close-pair
// contributions and the disk / diagonal terms:  apply: out = 1/2 p - R;  rhs:
// b = R - (eps/2) g.  One thread per output: the partials in ascending split order (8
// coalesced loads in flight; consecutive threads read consecutive rows), then the close
// pairs of the row in CSR order, their loads issued kFinBatch pairs at a time.
// (Tried: TMA bulk copies of each block's partial slices into shared memory — 1.9x slower.)
constexpr int kFinThreads = 256, kFinBatch = 2;
// Rows [r0, r0 + rows) of the operator (row sharding; r0 = 0, rows = M otherwise): part
// and out are [.][nsys][rows]; p and g are full vectors [nsys][ldp].
__global__ void __launch_bounds__(kFinThreads) mc_finish_kernel(int nsys, int64_t M, const double* __restrict__ smp,
                                                                const int32_t* __restrict__ rp,
                                                                const int32_t* __restrict__ col, KArr ka, double w,
                                                                const double2* part, int n_split,  // may alias out
                                                                const double2* __restrict__ p,
                                                                const double2* __restrict__ g, double eps,
                                                                double2* out,
                                                                const unsigned long long* __restrict__ skip,
                                                                int64_t r0, int64_t rows, int64_t ldp) {
  if (skip && *skip == 0ull) return;
  const int64_t il = blockIdx.x * (int64_t)kFinThreads + threadIdx.x;
  const int s = blockIdx.y;
  if (il >= rows) return;
  const int64_t i = r0 + il;
  const size_t q = (size_t)s * rows + il;
  const size_t stride = (size_t)nsys * rows;
  double ar = 0.0, ai = 0.0;
  for (int sp0 = 0; sp0 < n_split; sp0 += 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = sp0 + u < n_split ? part[(size_t)(sp0 + u) * stride + q] : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ar += v[u].x;
      ai += v[u].y;
    }
  }
  if (rp) {
    const double k = ka.k[s];
    const double xi = smp[i], yi = smp[M + i], zi = smp[2 * M + i];
    const int e1 = rp[i + 1];
    for (int e0 = rp[i]; e0 < e1; e0 += kFinBatch) {
      int32_t jj[kFinBatch];
#pragma unroll
      for (int u = 0; u < kFinBatch; ++u) jj[u] = e0 + u < e1 ? col[e0 + u] : -1;
      double dx[kFinBatch], dy[kFinBatch], dz[kFinBatch], dn[kFinBatch];
      double2 pv[kFinBatch], gv[kFinBatch];
#pragma unroll
      for (int u = 0; u < kFinBatch; ++u) {
        const int64_t j = jj[u] >= 0 ? jj[u] : i;
        dx[u] = smp[j] - xi;
        dy[u] = smp[M + j] - yi;
        dz[u] = smp[2 * M + j] - zi;
        if (p) {
          dn[u] = dx[u] * smp[3 * M + j] + dy[u] * smp[4 * M + j] + dz[u] * smp[5 * M + j];
          pv[u] = p[(size_t)s * ldp + j];
        }
        if (g) gv[u] = g[(size_t)s * ldp + j];
      }
#pragma unroll
      for (int u = 0; u < kFinBatch; ++u) {
        if (jj[u] < 0) continue;
        const double r = sqrt(dx[u] * dx[u] + dy[u] * dy[u] + dz[u] * dz[u]);
        float snf, csf;  // |kr| < 2 k eps: the fp32 phase is accurate to ~1e-7 absolute
        __sincosf((float)(k * r), &snf, &csf);
        const double sn = snf, cs = csf;
        const double t = w * nat::kInv4Pi / r;  // w G = t e^{ikr}
        if (p) {  // w p dG/dn_y = t dn/r^2 (ikr - 1) e^{ikr} p
          const double uu = t * dn[u] / (r * r);
          const double er = -cs - k * r * sn, ei = k * r * cs - sn;  // (ikr - 1) e^{ikr}
          ar += uu * (er * pv[u].x - ei * pv[u].y);
          ai += uu * (er * pv[u].y + ei * pv[u].x);
        }
        if (g) {  // - w g G
          ar -= t * (cs * gv[u].x - sn * gv[u].y);
          ai -= t * (cs * gv[u].y + sn * gv[u].x);
        }
      }
    }
  }
  if (p) {
    const double2 pi_ = p[(size_t)s * ldp + i];
    out[q] = make_double2(0.5 * pi_.x - ar, 0.5 * pi_.y - ai);
  } else {
    const double2 gi_ = g[(size_t)s * ldp + i];
    out[q] = make_double2(ar - 0.5 * eps * gi_.x, ai - 0.5 * eps * gi_.y);
  }
}

struct NearPairs {
  int32_t* rp = nullptr;   // [M+1]
  int32_t* col = nullptr;  // [cap]
  int* overflow = nullptr;
  int64_t cap = 0;
  float thr = 0.f;
  bool on = false;
};

int64_t near_cap(int64_t M) { return 64 * M + 1024; }

void carve_near(nat::Carver& c, NearPairs* np, int64_t M) {
  NearPairs t;
  t.cap = near_cap(M);
  t.rp = c.take<int32_t>(M + 1);
  t.col = c.take<int32_t>(t.cap);
  t.overflow = c.take<int>(1);
  if (np) *np = t;
}

// check = false: no read-back; the caller checks *np.overflow after its own final sync
// (the MC solve never stalls the host before its Krylov loop)
nat_status build_near(NearPairs& np, int64_t M, const double* smp, const double* center, double eps,
                      cudaStream_t s, bool check = true) {
  np.on = true;
  np.thr = (float)(4.0 * eps * eps);
  const double cx = center ? center[0] : 0.0, cy = center ? center[1] : 0.0, cz = center ? center[2] : 0.0;
  const unsigned grid = (unsigned)((M + kNW * kNRows - 1) / (kNW * kNRows));
  NAT_CUDA_TRY(cudaMemsetAsync(np.overflow, 0, sizeof(int), s));
  mc_near_kernel<false><<<grid, kNT, 0, s>>>(M, smp, cx, cy, cz, np.thr, np.rp, np.col, np.cap, np.overflow);
  scan32_kernel<<<1, 1024, 0, s>>>(np.rp, M, np.cap, np.overflow);
  mc_near_kernel<true><<<grid, kNT, 0, s>>>(M, smp, cx, cy, cz, np.thr, np.rp, np.col, np.cap, np.overflow);
  NAT_LAUNCH_CHECK();
  if (!check) return NAT_OK;
  int ov = 0;
  NAT_CUDA_TRY(cudaMemcpyAsync(&ov, np.overflow, sizeof(int), cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  if (ov) return nat::fail(NAT_ERR_WORKSPACE, "more than %lld close sample pairs", (long long)np.cap);
  return NAT_OK;
}

nat::RadInput self_input(int64_t M, const double* smp, int nsys, double w) {
  nat::RadInput in{};
  in.n_src = M;
  in.xyz = smp;
  in.nrm = smp + 3 * M;
  in.w = nullptr;
  in.w_const = w;
  in.n_modes = nsys;
  in.ldpg = M;
  in.center[0] = in.center[1] = in.center[2] = 0.0;
  return in;
}

// Target rows of an operator application (row sharding): rows [r0, r0 + rows) with their
// coordinates tgt [3][rows]; p / g are full vectors [nsys][ldp]; the output is [nsys][rows].
// Default: every row (r0 = 0, rows = M, tgt = the samples, ldp = M).
struct Rows {
  int64_t r0 = 0, rows = -1, ldp = -1;
  const double* tgt = nullptr;
};

// radiation kernel (partials kept) + one fused epilogue launch per 64 systems
nat_status finish_op(const nat::RadInput& in, nat_prec prec, int64_t M, const double* smp, int nsys,
                     const double* k, double w, double eps, const double2* p, const double2* g, double2* out,
                     void* ws, size_t ws_bytes, const NearPairs& np, cudaStream_t s, Rows rr = Rows{}) {
  const int64_t rows = rr.rows < 0 ? M : rr.rows, ldp = rr.ldp < 0 ? M : rr.ldp;
  const double* tgt = rr.tgt ? rr.tgt : smp;
  nat::RadPartials keep;
  nat_status st = nat::radiate_internal(in, prec, k, rows, tgt, out, ws, ws_bytes, true, s, &keep);
  if (st != NAT_OK) return st;
  KArr ka{};
  for (int q = 0; q < nsys && q < 64; ++q) ka.k[q] = k[q];
  mc_finish_kernel<<<dim3((unsigned)((rows + kFinThreads - 1) / kFinThreads), nsys), kFinThreads, 0, s>>>(
      nsys, M, smp, np.on ? np.rp : nullptr, np.on ? np.col : nullptr, ka, w, keep.part, keep.n_split, p, g, eps, out,
      in.skip, rr.r0, rows, ldp);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

nat_status mc_rhs_impl(nat_prec prec, int64_t M, const double* smp, int nsys, const double* k,
                       const double2* g, double w, double eps, double2* b, void* ws, size_t ws_bytes,
                       const double* center, const NearPairs& np, cudaStream_t s, Rows rr = Rows{}) {
  nat::RadInput in = self_input(M, smp, nsys, w);
  if (center)
    for (int d = 0; d < 3; ++d) in.center[d] = center[d];
  in.g = g;
  if (rr.ldp > 0) in.ldpg = rr.ldp;
  in.plan_lis = M;  // a row block sums its rows exactly as the full operator does
  in.self_r2 = np.on ? np.thr : 0.f;
  return finish_op(in, prec, M, smp, nsys, k, w, eps, nullptr, g, b, ws, ws_bytes, np, s, rr);
}

nat_status mc_apply_impl(nat_prec prec, int64_t M, const double* smp, int nsys, const double* k,
                         const double2* p, double w, double2* out, void* ws, size_t ws_bytes,
                         const double* center, const NearPairs& np, cudaStream_t s,
                         const unsigned long long* skip = nullptr, Rows rr = Rows{}) {
  nat::RadInput in = self_input(M, smp, nsys, w);
  if (center)
    for (int d = 0; d < 3; ++d) in.center[d] = center[d];
  in.p = p;
  in.skip = skip;
  if (rr.ldp > 0) in.ldpg = rr.ldp;
  in.plan_lis = M;  // a row block sums its rows exactly as the full operator does
  in.self_r2 = np.on ? np.thr : 0.f;
  return finish_op(in, prec, M, smp, nsys, k, w, 0.0, p, nullptr, out, ws, ws_bytes, np, s, rr);
}

// Disk radius and off-disk weight (readings R-eps, R-weight):
//   eps = sqrt(|Gamma| / (pi M)) unless the caller gives eps > 0,
//   w = (|Gamma| - pi eps^2) / (M - 1)   (w = 0 for M = 1: the single-sample row).
nat_status mc_eps_w(double area, int64_t M, double eps_in, double* eps, double* w) {
  NAT_REQUIRE(area > 0 && area < 1e300, "total_area = %g must be finite and > 0", area);
  *eps = eps_in > 0 ? eps_in : std::sqrt(area / (nat::kPi * (double)M));
  *w = M > 1 ? (area - nat::kPi * *eps * *eps) / (double)(M - 1) : 0.0;
  NAT_REQUIRE(*w >= 0, "eps = %g: the disk area pi eps^2 exceeds |Gamma| = %g", *eps, area);
  return NAT_OK;
}

// The fp32 solves keep their Krylov basis in fp32 (reading R-basis32; NAT_BASIS32=0: fp64).
bool basis32(nat_prec prec) {
  static const bool off = [] {
    const char* e = std::getenv("NAT_BASIS32");
    return e && e[0] == '0';
  }();
  return prec == NAT_FP32 && !off;
}

nat_status check_k(int n, const double* k) {
  NAT_REQUIRE(k, "k must be a host array");
  for (int m = 0; m < n; ++m)
    NAT_REQUIRE(k[m] >= 0.0 && k[m] < 1e300, "k[%d] = %g must be finite and >= 0", m, k[m]);
  return NAT_OK;
}

}  // namespace

extern "C" nat_status nat_mc_sample(const nat_mesh* mesh, const nat_geom* geom, int64_t M, uint64_t seed,
                                    uint64_t stream_id, double* samples, int32_t* sample_tri,
                                    nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(mesh && geom, "mesh and geom must be non-null");
  NAT_REQUIRE(M >= 1 && M < (1LL << 32), "M must be in [1, 2^32)");
  NAT_REQUIRE(geom->n_tri == mesh->n_tri && mesh->n_tri >= 1, "inconsistent n_tri");
  NAT_REQUIRE_DEV(mesh->vxyz);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->normal);
  NAT_REQUIRE_DEV(geom->area_cdf);
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(sample_tri);
  return nat::mc_sample_tagged(mesh, geom, M, seed, stream_id, 0u, samples, sample_tri, (cudaStream_t)stream);
}

nat_status nat::mc_sample_tagged(const nat_mesh* mesh, const nat_geom* geom, int64_t M, uint64_t seed,
                                 uint64_t stream_id, uint32_t tag, double* samples, int32_t* sample_tri,
                                 cudaStream_t stream) {
  mc_sample_kernel<<<(unsigned)((M + 255) / 256), 256, 0, stream>>>(
      M, seed, stream_id, tag, mesh->n_vert, mesh->n_tri, mesh->vxyz, mesh->tri, geom->normal, geom->area_cdf,
      samples, sample_tri);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

extern "C" nat_status nat_mc_check_coincident(int64_t M, const double* samples, int64_t* pair, void* ws,
                                              size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(M >= 1 && pair, "need M >= 1 and a host pair[2]");
  NAT_REQUIRE(ws_bytes >= 8, "workspace must hold 8 bytes");
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(ws);
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* best = (unsigned long long*)ws;
  init_best_kernel<<<1, 1, 0, s>>>(best);
  coincident_kernel<<<(unsigned)((M + kCT - 1) / kCT), kCT, 0, s>>>(M, samples, best);
  NAT_LAUNCH_CHECK();
  unsigned long long h = 0;
  NAT_CUDA_TRY(cudaMemcpyAsync(&h, best, 8, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  if (h == ~0ull) {
    pair[0] = pair[1] = -1;
    return NAT_OK;
  }
  pair[0] = (int64_t)(h >> 32);
  pair[1] = (int64_t)(h & 0xffffffffull);
  return nat::fail(NAT_ERR_SINGULAR, "coincident samples (%lld, %lld)", (long long)pair[0], (long long)pair[1]);
}

extern "C" nat_status nat_mc_gather_neumann(int n_sys, int64_t M, int64_t n_tri, const void* g_tri,
                                            const int32_t* sample_tri, void* g_out, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(n_sys >= 1 && M >= 1 && n_tri >= 1, "need n_sys, M, n_tri >= 1");
  NAT_REQUIRE_DEV(g_tri);
  NAT_REQUIRE_DEV(sample_tri);
  NAT_REQUIRE_DEV(g_out);
  for (int s0 = 0; s0 < n_sys; s0 += 65535) {
    const int nb = (n_sys - s0) < 65535 ? (n_sys - s0) : 65535;
    gather_g_kernel<<<dim3((unsigned)((M + 255) / 256), nb), 256, 0, (cudaStream_t)stream>>>(
        nb, M, n_tri, (const double2*)g_tri + (size_t)s0 * n_tri, sample_tri, (double2*)g_out + (size_t)s0 * M);
  }
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

extern "C" size_t nat_mc_op_workspace(nat_prec prec, int64_t M, int n_sys) {
  nat::Carver c(nullptr);
  carve_near(c, nullptr, M);
  c.take<char>(std::max(nat::radiate_ws_bytes(prec, M, n_sys, M, 1), nat::radiate_ws_bytes(prec, M, n_sys, M, 2)));
  return c.bytes();
}

namespace {
// Standalone a9 / a10 calls: near-pair list (fp32 path) + radiation scratch in ws.
nat_status op_setup(nat_prec prec, int64_t M, int n_sys, const double* smp, double eps, void* ws, size_t ws_bytes,
                    NearPairs& np, void** rad, size_t* rad_bytes, cudaStream_t s) {
  nat::Carver c(ws);
  carve_near(c, &np, M);
  *rad_bytes = std::max(nat::radiate_ws_bytes(prec, M, n_sys, M, 1), nat::radiate_ws_bytes(prec, M, n_sys, M, 2));
  *rad = c.take<char>(*rad_bytes);
  if (ws_bytes < c.bytes()) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, c.bytes());
  if (prec == NAT_FP32 && eps > 0) return build_near(np, M, smp, nullptr, eps, s);
  return NAT_OK;
}
}  // namespace

extern "C" nat_status nat_mc_rhs(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k,
                                 const void* g, double total_area, double eps_in, void* b, void* ws, size_t ws_bytes,
                                 nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(M >= 1 && n_sys >= 1, "need M >= 1 and n_sys >= 1");
  nat_status st = check_k(n_sys, k);
  if (st != NAT_OK) return st;
  double eps, w;
  st = mc_eps_w(total_area, M, eps_in, &eps, &w);
  if (st != NAT_OK) return st;
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(g);
  NAT_REQUIRE_DEV(b);
  NAT_REQUIRE_DEV(ws);
  NearPairs np;
  void* rad;
  size_t rad_bytes;
  st = op_setup(prec, M, n_sys, samples, eps, ws, ws_bytes, np, &rad, &rad_bytes, (cudaStream_t)stream);
  if (st != NAT_OK) return st;
  return mc_rhs_impl(prec, M, samples, n_sys, k, (const double2*)g, w, eps, (double2*)b, rad, rad_bytes,
                     nullptr, np, (cudaStream_t)stream);
}

extern "C" nat_status nat_mc_apply(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k,
                                   const void* p, double total_area, double eps_in, void* out, void* ws,
                                   size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(M >= 1 && n_sys >= 1, "need M >= 1 and n_sys >= 1");
  nat_status st = check_k(n_sys, k);
  if (st != NAT_OK) return st;
  double eps, w;
  st = mc_eps_w(total_area, M, eps_in, &eps, &w);
  if (st != NAT_OK) return st;
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(p);
  NAT_REQUIRE_DEV(out);
  NAT_REQUIRE_DEV(ws);
  NearPairs np;
  void* rad;
  size_t rad_bytes;
  st = op_setup(prec, M, n_sys, samples, eps, ws, ws_bytes, np, &rad, &rad_bytes, (cudaStream_t)stream);
  if (st != NAT_OK) return st;
  return mc_apply_impl(prec, M, samples, n_sys, k, (const double2*)p, w, (double2*)out, rad, rad_bytes, nullptr,
                       np, (cudaStream_t)stream);
}

namespace {
// tgt[d][i] = samples[d][r0 + i]: the target coordinates of a row block ([3][rows] SoA)
__global__ void copy_targets_kernel(int64_t M, const double* __restrict__ smp, int64_t r0, int64_t rows,
                                    double* __restrict__ tgt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (int d = 0; d < 3; ++d) tgt[(size_t)d * rows + i] = smp[(size_t)d * M + r0 + i];
}

struct SysIdx {  // system q of a compacted batch -> its slot in the full batch
  int idx[64];
};

// dst[sys(s)][r0 + i] = src[s][i] (a row block into full vectors of leading dimension ld;
// sys(s) = s, or ix.idx[s] for a compacted batch of the systems still iterating)
__global__ void place_rows_kernel(int64_t rows, int64_t r0, int64_t ld, const double2* __restrict__ src,
                                  double2* __restrict__ dst, const unsigned long long* __restrict__ skip,
                                  SysIdx ix, bool use_ix) {
  if (skip && *skip == 0ull) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  const int d = use_ix ? ix.idx[s] : s;
  if (i < rows) dst[(size_t)d * ld + r0 + i] = src[(size_t)s * rows + i];
}

// dst[s][:] = src[ix.idx[s]][:] over rows of length ld (compaction of the active systems)
__global__ void gather_sys_kernel(int64_t ld, SysIdx ix, const double2* __restrict__ src, double2* __restrict__ dst) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int s = blockIdx.y;
  if (j < ld) dst[(size_t)s * ld + j] = src[(size_t)ix.idx[s] * ld + j];
}
}  // namespace

extern "C" size_t nat_mc_rows_workspace(nat_prec prec, int64_t M, int n_sys, int64_t rows) {
  nat::Carver c(nullptr);
  carve_near(c, nullptr, M);
  c.take<double>((size_t)3 * (rows > 0 ? rows : 1));
  c.take<char>(std::max(nat::radiate_ws_bytes(prec, M, n_sys, rows, 1, M), nat::radiate_ws_bytes(prec, M, n_sys, rows, 2, M)));
  return c.bytes();
}

extern "C" nat_status nat_mc_apply_rows(nat_prec prec, int64_t M, const double* samples, int n_sys, const double* k,
                                        const void* p, double total_area, double eps_in, int64_t row_begin,
                                        int64_t row_end, void* out, void* ws, size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(M >= 1 && n_sys >= 1 && n_sys <= 64, "need M >= 1 and 1 <= n_sys <= 64");
  NAT_REQUIRE(0 <= row_begin && row_begin < row_end && row_end <= M, "bad row range");
  nat_status st = check_k(n_sys, k);
  if (st != NAT_OK) return st;
  double eps, w;
  st = mc_eps_w(total_area, M, eps_in, &eps, &w);
  if (st != NAT_OK) return st;
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(p);
  NAT_REQUIRE_DEV(out);
  NAT_REQUIRE_DEV(ws);
  const int64_t rows = row_end - row_begin;
  cudaStream_t s = (cudaStream_t)stream;
  nat::Carver c(ws);
  NearPairs np;
  carve_near(c, &np, M);
  double* tgt = c.take<double>((size_t)3 * rows);
  const size_t rad_bytes =
      std::max(nat::radiate_ws_bytes(prec, M, n_sys, rows, 1, M), nat::radiate_ws_bytes(prec, M, n_sys, rows, 2, M));
  void* rad = c.take<char>(rad_bytes);
  if (ws_bytes < c.bytes()) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, c.bytes());
  if (prec == NAT_FP32 && eps > 0) {
    st = build_near(np, M, samples, nullptr, eps, s);
    if (st != NAT_OK) return st;
  }
  copy_targets_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(M, samples, row_begin, rows, tgt);
  NAT_LAUNCH_CHECK();
  Rows rr;
  rr.r0 = row_begin;
  rr.rows = rows;
  rr.ldp = M;
  rr.tgt = tgt;
  return mc_apply_impl(prec, M, samples, n_sys, k, (const double2*)p, w, (double2*)out, rad, rad_bytes, nullptr, np,
                       s, nullptr, rr);
}

namespace {
constexpr int kMaxGroups = 4;
struct McGroupWs {   // one solve group: its Krylov state, operator workspace and compaction buffers
  nat::KrylovWs kw;
  void* rad;
  size_t rad_bytes;
  double2* tin;   // compacted operator input / output of the systems still iterating
  double2* tout;
};
struct McWs {
  unsigned long long* best;
  double2* gs;
  double2* b;
  NearPairs np;
  McGroupWs grp[kMaxGroups];
};

// Solve groups (NAT_MC_GROUPS or nat_mc_set_groups; default 2): the systems of a batch are
// split into G contiguous groups whose GMRES iterations run concurrently on G streams (one
// host thread each), so one group's latency-bound Krylov kernels overlap another group's
// operator application inside a single call.
std::atomic<int> g_mc_groups{0};
int mc_groups() {
  int v = g_mc_groups.load();
  if (v <= 0) {
    const char* e = std::getenv("NAT_MC_GROUPS");
    v = e ? std::max(1, std::min(kMaxGroups, std::atoi(e))) : 2;
    g_mc_groups.store(v);
  }
  return v;
}

// Persistent helper threads for the groups: libnat keeps per-thread pinned rings and events
// (gmres.cu HostSync), so the threads that run solves must outlive the calls.
class GroupPool {
 public:
  static GroupPool& get() {
    static GroupPool* p = new GroupPool();  // never destroyed: detached workers
    return *p;
  }
  std::future<nat_status> submit(std::function<nat_status()> f) {
    auto task = std::make_shared<std::packaged_task<nat_status()>>(std::move(f));
    std::future<nat_status> fut = task->get_future();
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push([task] { (*task)(); });
      while ((int)n_threads_ < (int)q_.size() + busy_ && n_threads_ < kMaxGroups) {
        std::thread([this] { loop(); }).detach();
        ++n_threads_;
      }
    }
    cv_.notify_one();
    return fut;
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        job = std::move(q_.front());
        q_.pop();
        ++busy_;
      }
      job();
      std::lock_guard<std::mutex> lk(mu_);
      --busy_;
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::queue<std::function<void()>> q_;
  int n_threads_ = 0, busy_ = 0;
};

// per-thread, per-device stream and event of a solve group
struct GroupStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev = nullptr;
};
GroupStream* group_stream() {
  thread_local std::map<int, GroupStream> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  GroupStream& g = per_dev[dev];
  if (!g.s) {
    if (cudaStreamCreateWithFlags(&g.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
  }
  return &g;
}

struct RowIdx {
  int idx[64];
};

// gather (dst[q] = src[idx[q]]) or scatter (dst[idx[q]] = src[q]) of [M]-rows
__global__ void copy_rows_kernel(RowIdx ix, int64_t M, const double2* __restrict__ src, double2* __restrict__ dst,
                                 bool gather) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (j >= M) return;
  if (gather)
    dst[(size_t)q * M + j] = src[(size_t)ix.idx[q] * M + j];
  else
    dst[(size_t)ix.idx[q] * M + j] = src[(size_t)q * M + j];
}

// smallest (i, j) with fp64 |y_i - y_j| < 1e-12 among the close pairs.
__global__ void coincident_near_kernel(int64_t M, const double* __restrict__ smp, const int32_t* __restrict__ rp,
                                       const int32_t* __restrict__ col, unsigned long long* best) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  for (int e = rp[i]; e < rp[i + 1]; ++e) {
    const int64_t j = col[e];
    const double dx = smp[j] - smp[i], dy = smp[M + j] - smp[M + i], dz = smp[2 * M + j] - smp[2 * M + i];
    if (sqrt(dx * dx + dy * dy + dz * dz) < 1e-12) {
      atomicMin(best, ((unsigned long long)i << 32) | (unsigned long long)j);
      return;
    }
  }
}

int group_size(int nb, int groups) { return (nb + groups - 1) / groups; }

size_t mc_carve(nat::Carver& c, McWs* w, nat_prec prec, int64_t M, int n_sys, int max_iter, int groups) {
  const int nb = n_sys < 64 ? n_sys : 64;
  const int G = std::max(1, std::min(groups, nb));
  const int nbg = group_size(nb, G);
  McWs t{};
  t.best = c.take<unsigned long long>(1);
  t.gs = c.take<double2>((size_t)nb * M);
  t.b = c.take<double2>((size_t)nb * M);
  carve_near(c, &t.np, M);
  for (int g = 0; g < G; ++g) {
    McGroupWs& q = t.grp[g];
    nat::krylov_workspace(nbg, M, M, max_iter, c, &q.kw);
    q.rad_bytes = nat::radiate_ws_bytes_upto(prec, M, nb, M);  // RHS (all nb systems) and the group's operator
    q.rad = g == 0 ? c.take<char>(q.rad_bytes) : nullptr;
    if (g > 0) {
      q.rad_bytes = nat::radiate_ws_bytes_upto(prec, M, nbg, M);
      q.rad = c.take<char>(q.rad_bytes);
    }
    q.tin = c.take<double2>((size_t)nbg * M);
    q.tout = c.take<double2>((size_t)nbg * M);
  }
  if (w) *w = t;
  return c.bytes();
}
}  // namespace

extern "C" size_t nat_mc_workspace(nat_prec prec, int64_t M, int n_sys, int max_iter) {
  if (max_iter <= 0) max_iter = 200;
  size_t b = 0;
  for (int g = 1; g <= kMaxGroups; ++g) {  // any group count the process may select
    nat::Carver c(nullptr);
    b = std::max(b, mc_carve(c, nullptr, prec, M, n_sys, max_iter, g));
  }
  return b;
}

extern "C" nat_status nat_mc_set_groups(int groups) {
  NAT_REQUIRE(groups >= 1 && groups <= kMaxGroups, "groups = %d must be in [1, %d]", groups, kMaxGroups);
  g_mc_groups.store(groups);
  return NAT_OK;
}

extern "C" nat_status nat_mc_surface_pressure(const nat_mesh* mesh, const nat_geom* geom, int n_sys,
                                              const double* k, const void* g_tri, const nat_mc_opts* opts,
                                              nat_prec prec, double tol, int max_iter, double* samples_out,
                                              int32_t* sample_tri_out, void* p_out, void* ws, size_t ws_bytes,
                                              nat_solve_info* info, nat_stream_t stream) {
  NAT_TRACE();
  auto t_start = std::chrono::steady_clock::now();
  NAT_REQUIRE(mesh && geom && opts, "mesh, geom and opts must be non-null");
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(n_sys >= 1, "n_sys must be >= 1");
  const int64_t M = opts->M;
  NAT_REQUIRE(M >= 1 && M < (1LL << 31), "M must be in [1, 2^31) (S:170)");
  NAT_REQUIRE(geom->total_area > 0, "geom->total_area must come from nat_mesh_prepare");
  nat_status st = check_k(n_sys, k);
  if (st != NAT_OK) return st;
  if (tol <= 0) tol = 1e-6;
  if (max_iter <= 0) max_iter = 200;
  NAT_REQUIRE_DEV(g_tri);
  NAT_REQUIRE_DEV(samples_out);
  NAT_REQUIRE_DEV(sample_tri_out);
  NAT_REQUIRE_DEV(p_out);
  NAT_REQUIRE_DEV(ws);
  nat::Carver c(ws);
  McWs w;
  const int groups = mc_groups();
  size_t need = mc_carve(c, &w, prec, M, n_sys, max_iter, groups);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  // a8: samples (or the caller's set, e.g. a host Poisson-disk set, enters unchanged)
  if (opts->samples_in) {
    NAT_REQUIRE_DEV(opts->samples_in);
    NAT_REQUIRE_DEV(opts->sample_tri_in);
    NAT_CUDA_TRY(cudaMemcpyAsync(samples_out, opts->samples_in, sizeof(double) * 6 * M, cudaMemcpyDeviceToDevice, s));
    NAT_CUDA_TRY(cudaMemcpyAsync(sample_tri_out, opts->sample_tri_in, sizeof(int32_t) * M, cudaMemcpyDeviceToDevice, s));
  } else {
    st = nat_mc_sample(mesh, geom, M, opts->seed, opts->stream_id, samples_out, sample_tri_out, stream);
    if (st != NAT_OK) return st;
  }
  // disk radius and off-disk weight (readings R-eps, R-weight)
  double eps, wgt;
  st = mc_eps_w(geom->total_area, M, opts->eps, &eps, &wgt);
  if (st != NAT_OK) return st;
  const double* cen = geom->center;
  if (M > 1) {
    // close pairs (fp32 r <= 2 eps); every coincident pair (fp64 r < 1e-12) is among them,
    // so the singularity check only scans this list.  Both checks are read back
    // after the solve (deferred): the host does not stall before the Krylov loop, and a
    // failed check still returns its error with no valid output.
    st = build_near(w.np, M, samples_out, cen, eps, s, false);
    if (st != NAT_OK) return st;
    init_best_kernel<<<1, 1, 0, s>>>(w.best);
    coincident_near_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(M, samples_out, w.np.rp, w.np.col, w.best);
    NAT_LAUNCH_CHECK();
    w.np.on = (prec == NAT_FP32);  // the fp64 kernel resolves close pairs itself
  }
  auto deferred = [&](nat_status solve_st) -> nat_status {
    if (M <= 1) return solve_st;
    unsigned long long hb = 0;
    int ov = 0;
    NAT_CUDA_TRY(cudaMemcpyAsync(&hb, w.best, 8, cudaMemcpyDeviceToHost, s));
    NAT_CUDA_TRY(cudaMemcpyAsync(&ov, w.np.overflow, sizeof(int), cudaMemcpyDeviceToHost, s));
    NAT_CUDA_TRY(cudaStreamSynchronize(s));
    if (hb != ~0ull)
      return nat::fail(NAT_ERR_SINGULAR, "coincident samples (%llu, %llu)", hb >> 32, hb & 0xffffffffull);
    if (ov) return nat::fail(NAT_ERR_WORKSPACE, "more than %lld close sample pairs", (long long)w.np.cap);
    return solve_st;
  };
  bool all_conv = true;
  for (int s0 = 0; s0 < n_sys; s0 += 64) {
    const int nb = (n_sys - s0) < 64 ? (n_sys - s0) : 64;
    gather_g_kernel<<<dim3((unsigned)((M + 255) / 256), nb), 256, 0, s>>>(
        nb, M, mesh->n_tri, (const double2*)g_tri + (size_t)s0 * mesh->n_tri, sample_tri_out, w.gs);
    NAT_LAUNCH_CHECK();
    st = mc_rhs_impl(prec, M, samples_out, nb, k + s0, w.gs, wgt, eps, w.b, w.grp[0].rad, w.grp[0].rad_bytes, cen,
                     w.np, s);
    if (st != NAT_OK) return deferred(st);
    const int G = std::max(1, std::min(groups, nb));
    const int nbg = group_size(nb, G);
    // group g: systems [g0, g0 + n) of the batch, its own Krylov state and operator workspace
    auto solve_group = [&, s0](int g, cudaStream_t gs_, std::vector<nat::KrylovResult>& res, double& t_op) -> nat_status {
      const int g0 = g * nbg, n = std::min(nbg, nb - g0);
      McGroupWs& q = w.grp[g];
      const double* kg = k + s0 + g0;
      const uint64_t all = n == 64 ? ~0ull : ((1ull << n) - 1);
      auto op = [&, n, kg, all](const double2* in, double2* out, uint64_t active, const unsigned long long* dmask,
                                cudaStream_t ss) -> nat_status {
        if ((active & all) == all)
          return mc_apply_impl(prec, M, samples_out, n, kg, in, wgt, out, q.rad, q.rad_bytes, cen, w.np, ss, dmask);
        // only the systems still iterating: gather them, apply, scatter back
        RowIdx ix{};
        double kc[64];
        int na = 0;
        for (int r = 0; r < n; ++r)
          if ((active >> r) & 1ull) {
            ix.idx[na] = r;
            kc[na++] = kg[r];
          }
        if (na == 0) return NAT_OK;
        const dim3 g2((unsigned)((M + 255) / 256), na);
        copy_rows_kernel<<<g2, 256, 0, ss>>>(ix, M, in, q.tin, true);
        nat_status r = mc_apply_impl(prec, M, samples_out, na, kc, q.tin, wgt, q.tout, q.rad, q.rad_bytes, cen, w.np,
                                     ss, dmask);
        if (r != NAT_OK) return r;
        copy_rows_kernel<<<g2, 256, 0, ss>>>(ix, M, q.tout, out, false);
        NAT_LAUNCH_CHECK();
        return NAT_OK;
      };
      return nat::gmres_batched(n, M, M, w.b + (size_t)g0 * M, (double2*)p_out + (size_t)(s0 + g0) * M, op, tol,
                                max_iter, q.kw, res, gs_, info ? &t_op : nullptr, basis32(prec));
    };
    std::vector<std::vector<nat::KrylovResult>> res(G);
    std::vector<double> t_op(G, 0.0);
    if (G == 1) {
      st = solve_group(0, s, res[0], t_op[0]);
      if (st != NAT_OK) return deferred(st);
    } else {
      // fork: every group stream waits for the right-hand side; join: s waits for every group
      GroupStream* mine = group_stream();
      if (!mine) return nat::fail(NAT_ERR_CUDA, "group stream: %s", cudaGetErrorString(cudaGetLastError()));
      NAT_CUDA_TRY(cudaEventRecord(mine->ev, s));
      cudaEvent_t fork = mine->ev;
      int dev = 0;
      NAT_CUDA_TRY(cudaGetDevice(&dev));
      std::vector<cudaEvent_t> joins(G, nullptr);
      auto run = [&, fork, dev](int g) -> nat_status {
        if (cudaSetDevice(dev) != cudaSuccess) return nat::fail(NAT_ERR_CUDA, "cudaSetDevice");
        GroupStream* gsx = group_stream();
        if (!gsx) return nat::fail(NAT_ERR_CUDA, "group stream");
        if (cudaStreamWaitEvent(gsx->s, fork, 0) != cudaSuccess) return nat::fail(NAT_ERR_CUDA, "stream wait");
        nat_status r = solve_group(g, gsx->s, res[g], t_op[g]);
        if (cudaEventRecord(gsx->ev, gsx->s) != cudaSuccess) return nat::fail(NAT_ERR_CUDA, "event record");
        joins[g] = gsx->ev;
        return r;
      };
      std::vector<std::future<nat_status>> fut;
      for (int g = 1; g < G; ++g) fut.push_back(GroupPool::get().submit([run, g] { return run(g); }));
      // group 0 on this thread, on a stream of its own (the fork event above stays on s)
      GroupStream* g0s = group_stream();
      nat_status st0 = NAT_OK;
      if (cudaStreamWaitEvent(g0s->s, fork, 0) != cudaSuccess) st0 = nat::fail(NAT_ERR_CUDA, "stream wait");
      if (st0 == NAT_OK) st0 = solve_group(0, g0s->s, res[0], t_op[0]);
      cudaEvent_t j0 = nullptr;
      if (cudaEventCreateWithFlags(&j0, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(j0, g0s->s);
        cudaStreamWaitEvent(s, j0, 0);
        cudaEventDestroy(j0);
      } else {
        cudaStreamSynchronize(g0s->s);
      }
      nat_status stg = st0;
      for (int g = 1; g < G; ++g) {
        nat_status r = fut[g - 1].get();
        if (joins[g]) NAT_CUDA_TRY(cudaStreamWaitEvent(s, joins[g], 0));
        if (stg == NAT_OK && r != NAT_OK) stg = r;
      }
      if (stg != NAT_OK) return deferred(stg);
    }
    for (int g = 0; g < G; ++g) {
      const int g0 = g * nbg, n = std::min(nbg, nb - g0);
      for (int q = 0; q < n; ++q) {
        all_conv = all_conv && res[g][q].converged;
        if (info) {
          info[s0 + g0 + q].iters = res[g][q].iters;
          info[s0 + g0 + q].converged = res[g][q].converged;
          info[s0 + g0 + q].rel_residual = res[g][q].rel_residual;
          info[s0 + g0 + q].t_matvec_s = t_op[g];
          info[s0 + g0 + q].t_comm_s = 0;
        }
      }
    }
  }
  st = deferred(NAT_OK);
  if (st != NAT_OK) return st;
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  double tt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  if (info)
    for (int q = 0; q < n_sys; ++q) {
      info[q].t_total_s = tt;
    }
  return all_conv ? NAT_OK : NAT_WARN_NOT_CONVERGED;
}

// ------------------------------------------------------------------------------------
// SURVEY §8(e) "MC, one large system": the same solve row-sharded across ranks — rank r
// owns sample rows [r ceil(M/g), ...) of the operator and the right-hand side; each
// operator application is followed by an in-place NCCL all-gather of every system's
// iterate (replicated Arnoldi, deterministic); every rank regenerates the identical
// Philox sample set (no sample communication).  comm == NULL: world 1.
// ------------------------------------------------------------------------------------
#include "nat_comm.cuh"

namespace {
struct McShardWs {
  unsigned long long* best;
  double2* gs;      // [nb][M]
  double2* bloc;    // [nb][rows]
  double2* bfull;   // [nb][ldv]
  double2* xfull;   // [nb][ldv]
  double2* oloc;    // [nb][rows]
  double* tgt;      // [3][rows]
  double2* tin;     // [nb][ldv] compacted operator input
  nat::KrylovWs kw;
  void* rad;
  size_t rad_bytes;
  NearPairs np;
};

size_t mc_shard_carve(nat::Carver& c, McShardWs* w, nat_prec prec, int64_t M, int n_sys, int max_iter, int world) {
  const int nb = n_sys < 64 ? n_sys : 64;
  const int64_t rpr = (M + world - 1) / world, ldv = rpr * world;
  McShardWs t;
  t.best = c.take<unsigned long long>(1);
  t.gs = c.take<double2>((size_t)nb * M);
  t.bloc = c.take<double2>((size_t)nb * rpr);
  t.bfull = c.take<double2>((size_t)nb * ldv);
  t.xfull = c.take<double2>((size_t)nb * ldv);
  t.oloc = c.take<double2>((size_t)nb * rpr);
  t.tgt = c.take<double>((size_t)3 * rpr);
  t.tin = c.take<double2>((size_t)nb * ldv);
  nat::krylov_workspace(nb, M, ldv, max_iter, c, &t.kw);
  // the operator shrinks to the active systems: the largest workspace over 1..nb systems
  t.rad_bytes = 0;
  for (int m = 1; m <= nb; ++m)
    t.rad_bytes = std::max(t.rad_bytes, std::max(nat::radiate_ws_bytes(prec, M, m, rpr, 1, M),
                                                 nat::radiate_ws_bytes(prec, M, m, rpr, 2, M)));
  t.rad = c.take<char>(t.rad_bytes);
  carve_near(c, &t.np, M);
  if (w) *w = t;
  return c.bytes();
}
}  // namespace

extern "C" size_t nat_mc_sharded_workspace(nat_prec prec, int64_t M, int n_sys, int max_iter, int world) {
  if (max_iter <= 0) max_iter = 200;
  if (world < 1) world = 1;
  nat::Carver c(nullptr);
  return mc_shard_carve(c, nullptr, prec, M, n_sys, max_iter, world);
}

extern "C" nat_status nat_mc_surface_pressure_sharded(nat_comm* comm, const nat_mesh* mesh, const nat_geom* geom,
                                                      int n_sys, const double* k, const void* g_tri,
                                                      const nat_mc_opts* opts, nat_prec prec, double tol,
                                                      int max_iter, double* samples_out, int32_t* sample_tri_out,
                                                      void* p_out, void* ws, size_t ws_bytes, nat_solve_info* info,
                                                      nat_stream_t stream) {
  NAT_TRACE();
  auto t_start = std::chrono::steady_clock::now();
  NAT_REQUIRE(mesh && geom && opts, "mesh, geom and opts must be non-null");
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(n_sys >= 1, "n_sys must be >= 1");
  const int64_t M = opts->M;
  NAT_REQUIRE(M >= 2 && M < (1LL << 31), "M must be in [2, 2^31) (S:170)");
  NAT_REQUIRE(geom->total_area > 0, "geom->total_area must come from nat_mesh_prepare");
  nat_status st = check_k(n_sys, k);
  if (st != NAT_OK) return st;
  if (tol <= 0) tol = 1e-6;
  if (max_iter <= 0) max_iter = 200;
  NAT_REQUIRE_DEV(g_tri);
  NAT_REQUIRE_DEV(samples_out);
  NAT_REQUIRE_DEV(sample_tri_out);
  NAT_REQUIRE_DEV(p_out);
  NAT_REQUIRE_DEV(ws);
  const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
  NAT_REQUIRE(world <= 64, "world size %d > 64", world);
  const int64_t rpr = (M + world - 1) / world, ldv = rpr * world;
  // every rank evaluates the same condition (no rank fails alone before a collective)
  NAT_REQUIRE((int64_t)(world - 1) * rpr < M, "the last of %d ranks owns no sample rows (M = %lld)", world,
              (long long)M);
  const int64_t r0 = std::min<int64_t>(M, (int64_t)rank * rpr), r1 = std::min<int64_t>(M, r0 + rpr);
  const int64_t rows = r1 - r0;
  nat::Carver c(ws);
  McShardWs w;
  const size_t need = mc_shard_carve(c, &w, prec, M, n_sys, max_iter, world);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  if (opts->samples_in) {
    NAT_REQUIRE_DEV(opts->samples_in);
    NAT_REQUIRE_DEV(opts->sample_tri_in);
    NAT_CUDA_TRY(cudaMemcpyAsync(samples_out, opts->samples_in, sizeof(double) * 6 * M, cudaMemcpyDeviceToDevice, s));
    NAT_CUDA_TRY(cudaMemcpyAsync(sample_tri_out, opts->sample_tri_in, sizeof(int32_t) * M, cudaMemcpyDeviceToDevice, s));
  } else {
    st = nat_mc_sample(mesh, geom, M, opts->seed, opts->stream_id, samples_out, sample_tri_out, stream);
    if (st != NAT_OK) return st;
  }
  double eps, wgt;
  st = mc_eps_w(geom->total_area, M, opts->eps, &eps, &wgt);
  if (st != NAT_OK) return st;
  const double* cen = geom->center;
  st = build_near(w.np, M, samples_out, cen, eps, s);
  if (st != NAT_OK) return st;
  init_best_kernel<<<1, 1, 0, s>>>(w.best);
  coincident_near_kernel<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(M, samples_out, w.np.rp, w.np.col, w.best);
  NAT_LAUNCH_CHECK();
  unsigned long long hb = 0;
  NAT_CUDA_TRY(cudaMemcpyAsync(&hb, w.best, 8, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  if (hb != ~0ull)
    return nat::fail(NAT_ERR_SINGULAR, "coincident samples (%llu, %llu)", hb >> 32, hb & 0xffffffffull);
  w.np.on = (prec == NAT_FP32);
  copy_targets_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(M, samples_out, r0, rows, w.tgt);
  NAT_LAUNCH_CHECK();
  Rows rr;
  rr.r0 = r0;
  rr.rows = rows;
  rr.tgt = w.tgt;
  int n_comm = 0;
  // one grouped all-gather of every system's iterate per operator application (every rank
  // issues the same groups in the same order); CUDA events around each for t_comm_s
  auto gather_all = [&](double2* full, int nb, cudaStream_t ss) -> nat_status {
    if (world == 1) return NAT_OK;
    std::vector<double*> bufs(nb);
    for (int q = 0; q < nb; ++q) bufs[q] = (double*)(full + (size_t)q * ldv);
    cudaEvent_t e0 = info ? nat::timing_event(1, 2 * n_comm) : nullptr;
    cudaEvent_t e1 = info ? nat::timing_event(1, 2 * n_comm + 1) : nullptr;
    if (e0 && e1) NAT_CUDA_TRY(cudaEventRecord(e0, ss));
    nat_status r = nat::allgather_inplace_many(comm, bufs.data(), nb, (size_t)rpr * 2, ss);
    if (r != NAT_OK) return r;
    if (e0 && e1) {
      NAT_CUDA_TRY(cudaEventRecord(e1, ss));
      ++n_comm;
    }
    return NAT_OK;
  };
  bool all_conv = true;
  for (int s0 = 0; s0 < n_sys; s0 += 64) {
    const int nb = (n_sys - s0) < 64 ? (n_sys - s0) : 64;
    gather_g_kernel<<<dim3((unsigned)((M + 255) / 256), nb), 256, 0, s>>>(
        nb, M, mesh->n_tri, (const double2*)g_tri + (size_t)s0 * mesh->n_tri, sample_tri_out, w.gs);
    NAT_LAUNCH_CHECK();
    rr.ldp = M;  // g: [nb][M]
    st = mc_rhs_impl(prec, M, samples_out, nb, k + s0, w.gs, wgt, eps, w.bloc, w.rad, w.rad_bytes, cen, w.np, s, rr);
    if (st != NAT_OK) return st;
    NAT_CUDA_TRY(cudaMemsetAsync(w.bfull, 0, sizeof(double2) * nb * ldv, s));
    place_rows_kernel<<<dim3((unsigned)((rows + 255) / 256), nb), 256, 0, s>>>(rows, r0, ldv, w.bloc, w.bfull,
                                                                               nullptr, SysIdx{}, false);
    NAT_LAUNCH_CHECK();
    st = gather_all(w.bfull, nb, s);
    if (st != NAT_OK) return st;
    const uint64_t all = nb == 64 ? ~0ull : ((1ull << nb) - 1);
    auto op = [&](const double2* in, double2* out, uint64_t active, const unsigned long long* dmask,
                  cudaStream_t ss) -> nat_status {
      Rows ro = rr;
      ro.ldp = ldv;  // the Krylov vectors: [nb][ldv]
      // only the systems still iterating (host mask, one iteration late): compact them
      SysIdx ix{};
      double kc[64];
      int na = 0;
      for (int q = 0; q < nb; ++q)
        if (((active & all) >> q) & 1ull) {
          ix.idx[na] = q;
          kc[na++] = k[s0 + q];
        }
      const bool compact = na < nb;
      if (na > 0) {
        const double2* src = in;
        if (compact) {
          gather_sys_kernel<<<dim3((unsigned)((ldv + 255) / 256), na), 256, 0, ss>>>(ldv, ix, in, w.tin);
          src = w.tin;
        }
        nat_status r = mc_apply_impl(prec, M, samples_out, na, compact ? kc : k + s0, src, wgt, w.oloc, w.rad,
                                     w.rad_bytes, cen, w.np, ss, dmask, ro);
        if (r != NAT_OK) return r;
        place_rows_kernel<<<dim3((unsigned)((rows + 255) / 256), na), 256, 0, ss>>>(rows, r0, ldv, w.oloc, out, dmask,
                                                                                   ix, compact);
        NAT_LAUNCH_CHECK();
      }
      return gather_all(out, nb, ss);
    };
    std::vector<nat::KrylovResult> res;
    double t_op = 0;
    st = nat::gmres_batched(nb, M, ldv, w.bfull, w.xfull, op, tol, max_iter, w.kw, res, s, info ? &t_op : nullptr,
                            basis32(prec));
    if (st != NAT_OK) return st;
    NAT_CUDA_TRY(cudaMemcpy2DAsync((double2*)p_out + (size_t)s0 * M, sizeof(double2) * M, w.xfull,
                                   sizeof(double2) * ldv, sizeof(double2) * M, nb, cudaMemcpyDeviceToDevice, s));
    for (int q = 0; q < nb; ++q) all_conv = all_conv && res[q].converged;
    if (info)
      for (int q = 0; q < nb; ++q) {
        info[s0 + q].iters = res[q].iters;
        info[s0 + q].converged = res[q].converged;
        info[s0 + q].rel_residual = res[q].rel_residual;
        info[s0 + q].t_matvec_s = t_op;
      }
  }
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  const double tt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  double t_comm = 0.0;
  for (int q = 0; q < n_comm; ++q) {
    float ms = 0.f;
    NAT_CUDA_TRY(cudaEventElapsedTime(&ms, nat::timing_event(1, 2 * q), nat::timing_event(1, 2 * q + 1)));
    t_comm += 1e-3 * ms;
  }
  if (info)
    for (int q = 0; q < n_sys; ++q) {
      info[q].t_total_s = tt;
      info[q].t_comm_s = t_comm;  // device time of the grouped all-gathers (all systems)
    }
  return all_conv ? NAT_OK : NAT_WARN_NOT_CONVERGED;
}
