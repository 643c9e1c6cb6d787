// Row a7 — unrestarted GMRES ("a tolerance of 1e-6 and a maximum of 200
// iterations"; reading R-gmres), batched over systems, plus the
// row-sharded dense-BEM driver nat_bem_solve (matvec -> NCCL all-gather -> replicated
// Arnoldi).  Arnoldi uses classical Gram-Schmidt applied twice (CGS2): two batched
// dot-product launches instead of j+1 dependent ones per iteration.  All reductions
// use fixed chunking (kKrylovChunk) and fixed in-block trees: deterministic, and
// identical on every rank and for every GPU count.  The Givens update, the convergence
// test and the back-substitution run on the device (one thread per system), so the host
// never stalls the GPU between iterations (krylov.cuh).
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>

#include <cooperative_groups.h>

#include "krylov.cuh"
#include "nat_comm.cuh"

namespace nat {
namespace {

constexpr int kT = 256;
constexpr int kRing = 4;  // pinned mask slots / events in flight
constexpr int kKU = 16;   // basis vectors loaded together by the update / combine kernels

__device__ __forceinline__ bool sys_on(uint64_t active, const unsigned long long* dmask, int s) {
  uint64_t a = active;
  if (dmask) a &= *dmask;
  return (a >> s) & 1ull;
}

__device__ __forceinline__ double2 block_reduce(double2 v, double2* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int q = 0; q < kT / 32; ++q) {
      s.x += sm[q].x;
      s.y += sm[q].y;
    }
  return s;
}

// Sum of p[0..cnt) by one warp: lane l takes l, l+32, ... (loads in flight together),
// then a fixed xor tree; every lane returns the total.  Deterministic.
__device__ __forceinline__ double2 warp_sum_partials(const double2* p, int cnt) {
  const int lane = threadIdx.x & 31;
  double2 t = make_double2(0.0, 0.0);
  for (int c = lane; c < cnt; c += 32) {
    const double2 v = __ldcg(&p[c]);
    t.x += v.x;
    t.y += v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
    t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
  }
  return t;
}

// Fixed-order sum of the nvec x nchunk partials of system s into h / h2 (one warp per
// vector):  mode 0: h = h2 = sum;  mode 1: h2 = sum, h += sum;  mode 2: h[s][slot] =
// (sqrt(Re sum), 0)
__device__ void finish_sums(const double2* __restrict__ part, int s, int nvec, int nchunk, int mp1, int mp2,
                            int mode, int slot, double2* __restrict__ h, double2* __restrict__ h2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (nchunk <= 32) {
    // one thread per vector, partials summed in chunk order with all loads in flight: a
    // single L2 round trip instead of one per group of 8 vectors (ncu r01: tail of dots)
    for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
      const double2* pk = part + ((size_t)s * mp1 + k) * nchunk;
      double2 v[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = c < nchunk ? __ldcg(&pk[c]) : make_double2(0.0, 0.0);
      double2 t = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        t.x += v[c].x;
        t.y += v[c].y;
      }
      if (mode == 0) {
        h[(size_t)s * mp2 + k] = t;
        h2[(size_t)s * mp2 + k] = t;
      } else if (mode == 1) {
        h2[(size_t)s * mp2 + k] = t;
        const double2 o = h[(size_t)s * mp2 + k];
        h[(size_t)s * mp2 + k] = make_double2(o.x + t.x, o.y + t.y);
      } else {
        h[(size_t)s * mp2 + slot] = make_double2(sqrt(t.x), 0.0);
      }
    }
    return;
  }
  for (int k = warp; k < nvec; k += nw) {
    const double2 t = warp_sum_partials(part + ((size_t)s * mp1 + k) * nchunk, nchunk);
    if (lane != 0) continue;
    if (mode == 0) {
      h[(size_t)s * mp2 + k] = t;
      h2[(size_t)s * mp2 + k] = t;
    } else if (mode == 1) {
      h2[(size_t)s * mp2 + k] = t;
      const double2 o = h[(size_t)s * mp2 + k];
      h[(size_t)s * mp2 + k] = make_double2(o.x + t.x, o.y + t.y);
    } else {
      h[(size_t)s * mp2 + slot] = make_double2(sqrt(t.x), 0.0);
    }
  }
}

// True for exactly one block of system s: the last one to finish (its partials are then
// all visible).  The counter is reset for the next launch.
__device__ bool last_block(unsigned* cnt, unsigned total, bool* flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(cnt, 1u);
    *flag = (prev == total - 1);
    if (*flag) *cnt = 0u;
  }
  __syncthreads();
  if (*flag) __threadfence();
  return *flag;
}

// part[s][k][c] = sum_{i in chunk c} conj(V_k[s][i]) w[s][i]; the last block of each
// system reduces the partials (fixed order) into h / h2 (finish_sums).
__global__ void __launch_bounds__(kT) dots_kernel(const double2* __restrict__ V, size_t vstride_k,
                                                 int64_t ldv, const double2* __restrict__ w, int64_t n,
                                                 int nvec, int nchunk, int mp1, uint64_t active,
                                                 const unsigned long long* __restrict__ dmask,
                                                 double2* __restrict__ part, int mp2, int mode, int slot,
                                                 double2* __restrict__ h, double2* __restrict__ h2,
                                                 unsigned* __restrict__ cnt) {
  __shared__ double2 sm[kT / 32];
  __shared__ bool flag;
  const int c = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  if (!sys_on(active, dmask, s)) return;
  const double2* v = V + k * vstride_k + (size_t)s * ldv;
  const double2* ww = w + (size_t)s * ldv;
  const int64_t i0 = (int64_t)c * kKrylovChunk;
  double2 acc = make_double2(0.0, 0.0);
  constexpr int U = kKrylovChunk / kT;
  double2 a[U], b[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * kT + threadIdx.x;
    a[u] = i < n ? v[i] : make_double2(0.0, 0.0);
    b[u] = i < n ? ww[i] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    acc.x += a[u].x * b[u].x + a[u].y * b[u].y;
    acc.y += a[u].x * b[u].y - a[u].y * b[u].x;
  }
  double2 r = block_reduce(acc, sm);
  if (threadIdx.x == 0) part[((size_t)s * mp1 + k) * nchunk + c] = r;
  if (last_block(&cnt[s], (unsigned)(nchunk * nvec), &flag))
    finish_sums(part, s, nvec, nchunk, mp1, mp2, mode, slot, h, h2);
}

// dst[s][i] = src[s][i] / h[s][slot]   (slot = norm); zero if the norm is 0
// With `publish` (host-mapped pinned word), block (0, 0) first copies the live mask there.
__global__ void scale_kernel(const double2* __restrict__ src, int64_t ldv, int64_t n, int mp2, int slot,
                             uint64_t active, const unsigned long long* __restrict__ dmask,
                             const double2* __restrict__ h, double2* __restrict__ dst,
                             volatile unsigned long long* publish) {
  const int s = blockIdx.y;
  if (publish && blockIdx.x == 0 && s == 0 && threadIdx.x == 0) {
    *publish = *dmask;
    __threadfence_system();
  }
  if (!sys_on(active, dmask, s)) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double nv = h[(size_t)s * mp2 + slot].x;
  double2 v = src[(size_t)s * ldv + i];
  dst[(size_t)s * ldv + i] = nv > 0 ? make_double2(v.x / nv, v.y / nv) : make_double2(0.0, 0.0);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cjmul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// beta = ||b|| (h[s][0]), gamma_0 = beta, k = 0; systems with b = 0 are done (x = 0,
// S:281), a non-finite norm is flagged.
__global__ void gm_init_kernel(int nsys, int mp1, int mp2, const double2* __restrict__ h, double2* __restrict__ gam,
                               DevSys* __restrict__ sys, unsigned long long* __restrict__ mask) {
  __shared__ unsigned long long bits;
  const int q = threadIdx.x;
  if (q == 0) bits = 0ull;
  __syncthreads();
  if (q < nsys) {
    const double beta = h[(size_t)q * mp2].x;
    DevSys S{beta, 0, 0};
    gam[(size_t)q * mp1] = make_double2(beta, 0.0);
    if (!isfinite(beta))
      S.flags = kSysNonFinite;
    else if (beta == 0.0)
      S.flags = kSysConverged;
    else
      atomicOr(&bits, 1ull << q);
    sys[q] = S;
  }
  __syncthreads();
  if (q == 0) *mask = bits;
}

// Givens state of the batched solve (device pointers) for the fused update kernel.
struct GivensArgs {
  int j, m, mp1, mp2;
  double tol;
  const double2* h;
  double2 *H, *cs, *sn, *gam;
  DevSys* sys;
  unsigned long long* mask;
};

// Arnoldi column j of system q, run by one whole block: apply the previous rotations,
// form the new one, update gamma and decide convergence (|gamma_{j+1}| <= tol beta, or
// breakdown) or the iteration cap; the mask bit is cleared when the system stops.  The
// column and the rotations are staged in shared memory (gsm: mp1 + 2m entries); one
// thread runs the sequential rotation chain.
__device__ void givens_block(const GivensArgs& g, int q, double2* gsm) {
  const int j = g.j, m = g.m, mp1 = g.mp1, tid = threadIdx.x, nt = blockDim.x;
  double2* col = gsm;
  double2* sc = gsm + mp1;
  double2* ss = sc + m;
  const double2* hq = g.h + (size_t)q * g.mp2;
  double2* c = g.cs + (size_t)q * m;
  double2* s = g.sn + (size_t)q * m;
  for (int i = tid; i <= j + 1; i += nt) col[i] = __ldcg(&hq[i]);
  for (int i = tid; i < j; i += nt) {
    sc[i] = c[i];
    ss[i] = s[i];
  }
  __syncthreads();
  if (tid == 0) {
    double2* gm = g.gam + (size_t)q * mp1;
    DevSys S = g.sys[q];
    S.k = j + 1;
    const double nrm = col[j + 1].x;
    if (!isfinite(nrm)) {
      S.flags |= kSysNonFinite;
      g.sys[q] = S;
      atomicAnd(g.mask, ~(1ull << q));
    } else {
      const bool breakdown = nrm == 0.0;
      // the rotation chain: the rotated entry i + 1 carries to step i + 1 in registers, the
      // original entries and the rotations of the next 8 steps are loaded ahead (the same
      // operations in the same order as one step at a time)
      double2 carry = col[0];
      for (int i0 = 0; i0 < j; i0 += 8) {
        double2 b[8], cc[8], sv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u < j ? i0 + u : j - 1;
          b[u] = col[i + 1];
          cc[u] = sc[i];
          sv[u] = ss[i];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (i0 + u >= j) break;
          const double2 hi = carry, hi1 = b[u];
          col[i0 + u] = cadd(cjmul(cc[u], hi), cjmul(sv[u], hi1));
          const double2 t = cmul(sv[u], hi);
          carry = cadd(make_double2(-t.x, -t.y), cmul(cc[u], hi1));
        }
      }
      col[j] = carry;
      const double2 a = col[j], bb = col[j + 1];
      const double den = sqrt((a.x * a.x + a.y * a.y) + (bb.x * bb.x + bb.y * bb.y));
      double2 cj = make_double2(1.0, 0.0), sj = make_double2(0.0, 0.0);
      if (den != 0.0) {
        cj = make_double2(a.x / den, a.y / den);
        sj = make_double2(bb.x / den, bb.y / den);
      }
      c[j] = cj;
      s[j] = sj;
      col[j] = cadd(cjmul(cj, a), cjmul(sj, bb));
      col[j + 1] = make_double2(0.0, 0.0);
      const double2 gj = gm[j];
      const double2 t = cmul(sj, gj);
      const double2 g1 = make_double2(-t.x, -t.y);
      gm[j + 1] = g1;
      gm[j] = cjmul(cj, gj);
      const bool stop_conv = hypot(g1.x, g1.y) <= g.tol * S.beta || breakdown;
      if (stop_conv) S.flags |= kSysConverged;
      g.sys[q] = S;
      if (stop_conv || j + 1 == m) atomicAnd(g.mask, ~(1ull << q));
    }
  }
  __syncthreads();
  double2* Hc = g.H + ((size_t)q * m + j) * mp1;
  for (int i = tid; i <= j + 1; i += nt) Hc[i] = col[i];
}

// w[s][i] = w_in[s][i] - sum_{k < nvec} h2[s][k] V_k[s][i] (w_in may be w); with norm_slot >= 0 also
// h[s][norm_slot] = ||w[s]|| (block partials, last block sums them in fixed order), and
// with `giv` that last block then runs the Givens step of system s (dynamic smem).
__global__ void __launch_bounds__(kT) update_kernel(const double2* __restrict__ V, size_t vstride_k, int64_t ldv,
                                                   int64_t n, int nvec, int mp2, uint64_t active,
                                                   const unsigned long long* __restrict__ dmask,
                                                   const double2* __restrict__ h2, const double2* w_in,
                                                   double2* w, int norm_slot, double2* __restrict__ h,
                                                   double2* __restrict__ npart, unsigned* __restrict__ cnt,
                                                   bool giv, GivensArgs ga) {
  extern __shared__ double2 gsm[];
  __shared__ double2 sm[kT / 32];
  __shared__ bool flag;
  const int s = blockIdx.y;
  if (!sys_on(active, dmask, s)) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double2 o = make_double2(0.0, 0.0);
  if (i < n) {
    // groups of kKU basis vectors: their loads are issued together (a long basis is
    // otherwise one dependent L2 round trip per vector), summed in ascending k
    double2 acc = make_double2(0.0, 0.0);
    const double2* vi = V + (size_t)s * ldv + i;
    for (int k0 = 0; k0 < nvec; k0 += kKU) {
      double2 v[kKU], c[kKU];
#pragma unroll
      for (int u = 0; u < kKU; ++u) {
        const int k = k0 + u;
        v[u] = k < nvec ? vi[k * vstride_k] : make_double2(0.0, 0.0);
        c[u] = k < nvec ? h2[(size_t)s * mp2 + k] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kKU; ++u) {
        if (k0 + u < nvec) {
          acc.x += c[u].x * v[u].x - c[u].y * v[u].y;
          acc.y += c[u].x * v[u].y + c[u].y * v[u].x;
        }
      }
    }
    o = w_in[(size_t)s * ldv + i];
    o = make_double2(o.x - acc.x, o.y - acc.y);
    w[(size_t)s * ldv + i] = o;
  }
  if (norm_slot < 0) return;
  const double2 r = block_reduce(make_double2(o.x * o.x + o.y * o.y, 0.0), sm);
  if (threadIdx.x == 0) npart[(size_t)s * gridDim.x + blockIdx.x] = r;
  if (last_block(&cnt[s], gridDim.x, &flag)) {
    if (threadIdx.x < 32) {
      const double t = warp_sum_partials(npart + (size_t)s * gridDim.x, (int)gridDim.x).x;
      if (threadIdx.x == 0) h[(size_t)s * mp2 + norm_slot] = make_double2(sqrt(t), 0.0);
    }
    if (giv) {
      __syncthreads();
      givens_block(ga, s, gsm);
    }
  }
}

// y = R^{-1} gamma (k x k upper triangle of the rotated Hessenberg matrix), one block
// per system, column-oriented: y_i = r_i / R_ii, then r_t -= R_ti y_i for t < i in
// parallel.  The triangle is staged in shared memory (packed by columns) when it fits.
constexpr int kBackT = 256;
constexpr int kBackSmemMax = 200 * 1024;
__global__ void __launch_bounds__(kBackT) backsolve_kernel(int m, int mp1, const double2* __restrict__ H,
                                                           const double2* __restrict__ gam,
                                                           const DevSys* __restrict__ sys,
                                                           double2* __restrict__ y, int smem_bytes) {
  extern __shared__ double2 bsm[];  // r[m], y[m], packed triangle (staged)
  const int q = blockIdx.x, tid = threadIdx.x;
  const int k = (sys[q].flags & kSysNonFinite) ? 0 : sys[q].k;
  const double2* Hq = H + (size_t)q * m * mp1;
  double2* r = bsm;
  double2* yy = bsm + m;
  double2* tri = bsm + 2 * m;
  const bool staged = sizeof(double2) * (2 * (size_t)m + (size_t)k * (k + 1) / 2) <= (size_t)smem_bytes;
  for (int i = tid; i < k; i += kBackT) r[i] = gam[(size_t)q * mp1 + i];
  if (staged)
    for (int i = 0; i < k; ++i)
      for (int t = tid; t <= i; t += kBackT) tri[i * (i + 1) / 2 + t] = Hq[(size_t)i * mp1 + t];
  __syncthreads();
  for (int i = k - 1; i >= 0; --i) {
    if (tid == 0) yy[i] = cdiv(r[i], staged ? tri[i * (i + 1) / 2 + i] : Hq[(size_t)i * mp1 + i]);
    __syncthreads();
    const double2 yi = yy[i];
    for (int t = tid; t < i; t += kBackT) {
      const double2 hv = staged ? tri[i * (i + 1) / 2 + t] : Hq[(size_t)i * mp1 + t];
      const double2 p = cmul(hv, yi);
      r[t] = make_double2(r[t].x - p.x, r[t].y - p.y);
    }
    __syncthreads();
  }
  for (int i = tid; i < k; i += kBackT) y[(size_t)q * m + i] = yy[i];
}

// x[s][i] = sum_{k < k_s} y[s][k] V_k[s][i] and, from the operator products W_k = A V_k
// saved during the iteration, r[s][i] = b[s][i] - sum_k y[s][k] W_k[s][i] = (b - A x)[s][i]
// (linearity: the true residual without another operator application).
__global__ void combine_kernel(const double2* __restrict__ V, const double2* __restrict__ W, size_t vstride_k,
                               int64_t ldv, int64_t n, int m, const double2* __restrict__ y,
                               const DevSys* __restrict__ sys, const double2* __restrict__ b,
                               double2* __restrict__ x, double2* __restrict__ r) {
  const int s = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int kmax = (sys[s].flags & kSysNonFinite) ? 0 : sys[s].k;
  double2 acc = make_double2(0.0, 0.0), ax = make_double2(0.0, 0.0);
  const size_t off = (size_t)s * ldv + i;
  for (int k0 = 0; k0 < kmax; k0 += kKU) {  // loads of kKU vectors in flight, ascending sums
    double2 c[kKU], v[kKU], u[kKU];
#pragma unroll
    for (int q = 0; q < kKU; ++q) {
      const int k = k0 + q;
      const bool on = k < kmax;
      c[q] = on ? y[(size_t)s * m + k] : make_double2(0.0, 0.0);
      v[q] = on ? V[k * vstride_k + off] : make_double2(0.0, 0.0);
      u[q] = on ? W[k * vstride_k + off] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < kKU; ++q) {
      if (k0 + q < kmax) {
        acc.x += c[q].x * v[q].x - c[q].y * v[q].y;
        acc.y += c[q].x * v[q].y + c[q].y * v[q].x;
        ax.x += c[q].x * u[q].x - c[q].y * u[q].y;
        ax.y += c[q].x * u[q].y + c[q].y * u[q].x;
      }
    }
  }
  x[(size_t)s * ldv + i] = acc;
  const double2 bb = b[(size_t)s * ldv + i];
  r[(size_t)s * ldv + i] = make_double2(bb.x - ax.x, bb.y - ax.y);
}

// ------------------------------------------------------------------------------------
// Fused Arnoldi step for short vectors (n <= CL x 2048; the MC systems, M = 2048-10,000):
// one thread-block cluster of CL CTAs per system runs the whole CGS2 iteration after the
// operator product — both projection passes (dots + update), the norm, the Givens step of
// the system and the scaling of the new basis vector — in ONE launch.  CTA c owns rows
// [c rpc, (c+1) rpc) of the system; the per-CTA partial dot products are exchanged through
// distributed shared memory and summed by every CTA in CTA order (deterministic, the same
// in every CTA).  A cluster touches its system's basis slice four times within a few
// microseconds, so three of the four passes hit L2 (the multi-kernel path streams the
// whole batched basis from HBM in every pass).  Requesting kFusedSmem bytes of shared
// memory caps residency at one CTA per SM, which keeps the basis slices of the clusters in
// flight (~18 systems) inside the 126 MB L2.
// ------------------------------------------------------------------------------------
constexpr int kFusedMaxRT = 8;                 // rows per thread (n <= CL x 256 x 8)
constexpr int kFusedSmem = 120 * 1024;         // residency cap (1 CTA / SM)

// Shape of the fused Arnoldi step, process-wide: nat_krylov_config() sets it at run time;
// until then the NAT_FUSED_CL / NAT_FUSED_NTH / NAT_FUSED_SMEM_KB / NAT_FUSED_NARROW
// environment variables (A/B runs) or the defaults (4 CTAs, 512 threads, 120 KB) apply.
struct KrylovConfig {
  int cl, nth, smem_kb;
};
std::atomic<int> g_kcfg_cl{0}, g_kcfg_nth{0}, g_kcfg_smem{-1};
KrylovConfig krylov_config() {
  if (g_kcfg_cl.load() == 0) {
    const char* e = std::getenv("NAT_FUSED_CL");
    const int cl = e ? std::atoi(e) : 4;
    const char* t = std::getenv("NAT_FUSED_NTH");
    const char* nw = std::getenv("NAT_FUSED_NARROW");
    const int nth = (t && std::atoi(t) == 256) ? 256 : (nw && nw[0] == '0') ? 768 : 512;
    const char* sm = std::getenv("NAT_FUSED_SMEM_KB");
    int expected = -1;
    g_kcfg_smem.compare_exchange_strong(expected, sm ? std::max(0, std::atoi(sm)) : kFusedSmem / 1024);
    int z = 0;
    g_kcfg_nth.compare_exchange_strong(z, nth);
    z = 0;
    g_kcfg_cl.compare_exchange_strong(z, cl == 8 ? 8 : cl == 2 ? 2 : 4);
  }
  return KrylovConfig{g_kcfg_cl.load(), g_kcfg_nth.load(), g_kcfg_smem.load()};
}

// Threads: NTH = KG x 256.  Dots: NTH / 32 warps, each two basis vectors at a time (16
// loads of 16 B in flight per lane).  Update: group g (256 threads, RT rows each) sums the
// basis vectors k = g, g + KG, ... in ascending order; group 0 adds the KG partial sums in
// group order (deterministic) and keeps w in registers.
template <int RT, int NTH, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NTH, 1)
    arnoldi_fused_kernel(const double2* __restrict__ V, size_t vstride, int64_t ldv, int64_t n, int64_t rpc,
                         const double2* __restrict__ Wj, double2* __restrict__ Vnext, uint64_t active,
                         GivensArgs ga) {
  namespace cg = cooperative_groups;
  constexpr int KG = NTH / kT, NW = NTH / 32;
  // [rpc] w | [2][mp1] partials | [mp1] h | [mp1] pass-1 coefficients | [KG-1][rpc] update partials
  extern __shared__ __align__(16) double2 fsm[];
  __shared__ double red[kT / 32];
  __shared__ double nrm_part, nrm_all;
  cg::cluster_group cl = cg::this_cluster();
  const int s = blockIdx.y;
  const int c = (int)cl.block_rank();
  const int j = ga.j, mp1 = ga.mp1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / kT, tr = tid % kT;
  // whole clusters skip (the mask bit of system s only changes in the Givens step after this)
  if (!sys_on(active, ga.mask, s)) return;
  double2* wsh = fsm;
  double2* hp = fsm + rpc;         // [2][mp1]
  double2* hs = hp + 2 * mp1;      // [mp1]
  double2* hc1 = hs + mp1;         // [mp1]
  double2* upd = hc1 + mp1;        // [KG-1][rpc]
  const int64_t r0 = (int64_t)c * rpc;
  const int rows = (int)max((int64_t)0, min(rpc, n - r0));
  const double2* Vs = V + (size_t)s * ldv + r0;
  double2 w[RT];
  if (grp == 0) {
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      w[q] = r < rows ? Wj[(size_t)s * ldv + r0 + r] : make_double2(0.0, 0.0);
      if (r < rows) wsh[r] = w[q];
    }
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double2* part = hp + pass * mp1;
    for (int k = warp; k <= j; k += 2 * NW) {
      const int k2 = k + NW;
      const double2* vk = Vs + (size_t)k * vstride;
      const double2* vk2 = Vs + (size_t)(k2 <= j ? k2 : k) * vstride;
      double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
      for (int r0l = 0; r0l < rows; r0l += 32 * 8) {
        double2 v[8], v2[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = r0l + q * 32 + lane;
          v[q] = r < rows ? __ldcg(&vk[r]) : make_double2(0.0, 0.0);
          v2[q] = r < rows ? __ldcg(&vk2[r]) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = r0l + q * 32 + lane;
          const double2 u = r < rows ? wsh[r] : make_double2(0.0, 0.0);
          ax += v[q].x * u.x + v[q].y * u.y;
          ay += v[q].x * u.y - v[q].y * u.x;
          bx += v2[q].x * u.x + v2[q].y * u.y;
          by += v2[q].x * u.y - v2[q].y * u.x;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, o);
        ay += __shfl_xor_sync(0xffffffffu, ay, o);
        bx += __shfl_xor_sync(0xffffffffu, bx, o);
        by += __shfl_xor_sync(0xffffffffu, by, o);
      }
      if (lane == 0) {
        part[k] = make_double2(ax, ay);
        if (k2 <= j) part[k2] = make_double2(bx, by);
      }
    }
    cl.sync();
    // this pass's coefficients = sum over the cluster's CTAs in rank order (the same in
    // every CTA); pass 0 keeps them in hp[1] (its partial slot is free until pass 1)
    double2* hc = pass == 0 ? hp + mp1 : hc1;
    for (int k = tid; k <= j; k += NTH) {
      double2 t = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const double2 p = cl.map_shared_rank(part, q)[k];
        t.x += p.x;
        t.y += p.y;
      }
      hs[k] = pass == 0 ? t : make_double2(hs[k].x + t.x, hs[k].y + t.y);
      hc[k] = t;
    }
    __syncthreads();
    // w_i -= sum_k hc[k] V_k[i]: group g takes k = g, g + KG, ... (8 loads in flight)
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      if (r >= rows) continue;
      double2 acc = make_double2(0.0, 0.0);
      const double2* vi = Vs + r;
      for (int k0 = grp; k0 <= j; k0 += 8 * KG) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k0 + u * KG;
          v[u] = k <= j ? __ldcg(&vi[(size_t)k * vstride]) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k0 + u * KG;
          const double2 cc = k <= j ? hc[k] : make_double2(0.0, 0.0);
          acc.x += cc.x * v[u].x - cc.y * v[u].y;
          acc.y += cc.x * v[u].y + cc.y * v[u].x;
        }
      }
      if (grp > 0) upd[(size_t)(grp - 1) * rpc + r] = acc;
      else w[q] = acc;  // group 0's partial, combined below
    }
    __syncthreads();
    if (grp == 0) {
#pragma unroll
      for (int q = 0; q < RT; ++q) {
        const int r = tr + q * kT;
        if (r >= rows) continue;
        double2 acc = w[q];
#pragma unroll
        for (int g = 1; g < KG; ++g) {
          const double2 u = upd[(size_t)(g - 1) * rpc + r];
          acc.x += u.x;
          acc.y += u.y;
        }
        const double2 wo = wsh[r];
        w[q] = make_double2(wo.x - acc.x, wo.y - acc.y);
      }
    }
    if (pass == 0) {
      // pass 1 writes its partials into hp[1] (which held the pass-0 coefficients) only
      // after every CTA of the cluster is done with its pass-0 update
      cl.sync();
      if (grp == 0) {
#pragma unroll
        for (int q = 0; q < RT; ++q) {
          const int r = tr + q * kT;
          if (r < rows) wsh[r] = w[q];
        }
      }
      __syncthreads();
    }
  }
  // ||w||^2: group-0 partial, cluster sum in rank order
  if (grp == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < RT; ++q) t += w[q].x * w[q].x + w[q].y * w[q].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[warp] = t;
  }
  __syncthreads();
  if (tid == 0) {
    double b = 0.0;
    for (int q = 0; q < kT / 32; ++q) b += red[q];
    nrm_part = b;
  }
  cl.sync();
  if (tid == 0) {
    double a = 0.0;
    for (int q = 0; q < CL; ++q) a += *cl.map_shared_rank(&nrm_part, q);
    nrm_all = sqrt(a);
  }
  __syncthreads();
  const double nv = nrm_all;
  if (grp == 0) {  // V_{j+1} = w / ||w|| (zero on breakdown, as scale_kernel)
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      if (r < rows)
        Vnext[(size_t)s * ldv + r0 + r] = nv > 0 ? make_double2(w[q].x / nv, w[q].y / nv) : make_double2(0.0, 0.0);
    }
  }
  if (c == 0) {  // the Hessenberg column of system s (its Givens step: givens_kernel)
    double2* hq = const_cast<double2*>(ga.h) + (size_t)s * ga.mp2;
    for (int k = tid; k <= j; k += NTH) hq[k] = hs[k];
    if (tid == 0) hq[j + 1] = make_double2(nv, 0.0);
  }
  cl.sync();  // no CTA exits while another may still read its shared memory
}

// Fused Arnoldi step over a basis stored as TB (double2, or float2: the fp32 solves,
// reading R-basis32 of DESIGN.md — the basis vectors are rounded to fp32 once when they
// are formed, and the operator, the dots, the updates and x = V y all use those rounded
// vectors, held exactly in fp64 in V and in fp32 in Vb; every product and sum is fp64).
// Same CTA / cluster structure and summation orders as arnoldi_fused_kernel; the loops
// keep more loads in flight per round trip: dots take UD rows per lane of two vectors at
// once (a CTA's whole 512-row slice in one round for float2), updates load U basis
// entries for each of the RT rows of a thread together.
template <typename TB>
__device__ __forceinline__ double2 to_d2(TB v) {
  return make_double2((double)v.x, (double)v.y);
}
template <typename TB>
__device__ __forceinline__ TB zero_tb() {
  TB v;
  v.x = 0;
  v.y = 0;
  return v;
}

template <typename TB, int RT, int NTH, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NTH, NTH <= 256 ? 2 : 1)
    arnoldi_fused_v2_kernel(const TB* __restrict__ Vb, size_t vstride, int64_t ldv, int64_t n, int64_t rpc,
                            const double2* __restrict__ Wj, double2* Vnext, TB* Vbnext,
                            uint64_t active, GivensArgs ga) {
  namespace cg = cooperative_groups;
  constexpr int KG = NTH / kT, NW = NTH / 32;
  constexpr int UD = sizeof(TB) == 8 ? 16 : 8;   // rows per lane per dot round
  constexpr int U0 = 16 / RT;
  constexpr int U = U0 > 0 ? U0 : 1;             // basis vectors per update round (x RT rows)
  extern __shared__ __align__(16) double2 fsm[];
  __shared__ double red[kT / 32];
  __shared__ double nrm_part, nrm_all;
  cg::cluster_group cl = cg::this_cluster();
  const int s = blockIdx.y;
  const int c = (int)cl.block_rank();
  const int j = ga.j, mp1 = ga.mp1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = tid / kT, tr = tid % kT;
  if (!sys_on(active, ga.mask, s)) return;
  double2* wsh = fsm;
  double2* hp = fsm + rpc;         // [2][mp1]
  double2* hs = hp + 2 * mp1;      // [mp1]
  double2* hc1 = hs + mp1;         // [mp1]
  double2* upd = hc1 + mp1;        // [KG-1][rpc]
  const int64_t r0 = (int64_t)c * rpc;
  const int rows = (int)max((int64_t)0, min(rpc, n - r0));
  const TB* Vs = Vb + (size_t)s * ldv + r0;
  double2 w[RT];
  if (grp == 0) {
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      w[q] = r < rows ? Wj[(size_t)s * ldv + r0 + r] : make_double2(0.0, 0.0);
      if (r < rows) wsh[r] = w[q];
    }
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double2* part = hp + pass * mp1;
    for (int k = warp; k <= j; k += 2 * NW) {
      const int k2 = k + NW;
      const TB* vk = Vs + (size_t)k * vstride;
      const TB* vk2 = Vs + (size_t)(k2 <= j ? k2 : k) * vstride;
      double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
      for (int r0l = 0; r0l < rows; r0l += 32 * UD) {
        TB v[UD], v2[UD];  // raw basis entries in flight, widened at use
#pragma unroll
        for (int q = 0; q < UD; ++q) {
          const int r = r0l + q * 32 + lane;
          v[q] = r < rows ? __ldcg(&vk[r]) : zero_tb<TB>();
          v2[q] = r < rows ? __ldcg(&vk2[r]) : zero_tb<TB>();
        }
#pragma unroll
        for (int q = 0; q < UD; ++q) {
          const int r = r0l + q * 32 + lane;
          const double2 u = r < rows ? wsh[r] : make_double2(0.0, 0.0);
          const double2 a = to_d2(v[q]), b = to_d2(v2[q]);
          ax += a.x * u.x + a.y * u.y;
          ay += a.x * u.y - a.y * u.x;
          bx += b.x * u.x + b.y * u.y;
          by += b.x * u.y - b.y * u.x;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        ax += __shfl_xor_sync(0xffffffffu, ax, o);
        ay += __shfl_xor_sync(0xffffffffu, ay, o);
        bx += __shfl_xor_sync(0xffffffffu, bx, o);
        by += __shfl_xor_sync(0xffffffffu, by, o);
      }
      if (lane == 0) {
        part[k] = make_double2(ax, ay);
        if (k2 <= j) part[k2] = make_double2(bx, by);
      }
    }
    cl.sync();
    double2* hc = pass == 0 ? hp + mp1 : hc1;
    for (int k = tid; k <= j; k += NTH) {
      double2 t = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const double2 p = cl.map_shared_rank(part, q)[k];
        t.x += p.x;
        t.y += p.y;
      }
      hs[k] = pass == 0 ? t : make_double2(hs[k].x + t.x, hs[k].y + t.y);
      hc[k] = t;
    }
    __syncthreads();
    // w_i -= sum_k hc[k] V_k[i]: group g takes k = g, g + KG, ... (RT x U loads in flight)
    double2 acc[RT];
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[q] = make_double2(0.0, 0.0);
    for (int k0 = grp; k0 <= j; k0 += U * KG) {
      TB v[RT][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * KG;
#pragma unroll
        for (int q = 0; q < RT; ++q) {
          const int r = tr + q * kT;
          v[q][u] = (k <= j && r < rows) ? __ldcg(&Vs[(size_t)k * vstride + r]) : zero_tb<TB>();
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u * KG;
        const double2 cc = k <= j ? hc[k] : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < RT; ++q) {
          const double2 a = to_d2(v[q][u]);
          acc[q].x += cc.x * a.x - cc.y * a.y;
          acc[q].y += cc.x * a.y + cc.y * a.x;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      if (r >= rows) continue;
      if (grp > 0) upd[(size_t)(grp - 1) * rpc + r] = acc[q];
      else w[q] = acc[q];
    }
    __syncthreads();
    if (grp == 0) {
#pragma unroll
      for (int q = 0; q < RT; ++q) {
        const int r = tr + q * kT;
        if (r >= rows) continue;
        double2 a = w[q];
#pragma unroll
        for (int g = 1; g < KG; ++g) {
          const double2 u = upd[(size_t)(g - 1) * rpc + r];
          a.x += u.x;
          a.y += u.y;
        }
        const double2 wo = wsh[r];
        w[q] = make_double2(wo.x - a.x, wo.y - a.y);
      }
    }
    if (pass == 0) {
      cl.sync();
      if (grp == 0) {
#pragma unroll
        for (int q = 0; q < RT; ++q) {
          const int r = tr + q * kT;
          if (r < rows) wsh[r] = w[q];
        }
      }
      __syncthreads();
    }
  }
  if (grp == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < RT; ++q) t += w[q].x * w[q].x + w[q].y * w[q].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[warp] = t;
  }
  __syncthreads();
  if (tid == 0) {
    double b = 0.0;
    for (int q = 0; q < kT / 32; ++q) b += red[q];
    nrm_part = b;
  }
  cl.sync();
  if (tid == 0) {
    double a = 0.0;
    for (int q = 0; q < CL; ++q) a += *cl.map_shared_rank(&nrm_part, q);
    nrm_all = sqrt(a);
  }
  __syncthreads();
  const double nv = nrm_all;
  if (grp == 0) {  // V_{j+1} = w / ||w|| (zero on breakdown), rounded to TB; V holds it exactly
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      const int r = tr + q * kT;
      if (r >= rows) continue;
      double2 v = nv > 0 ? make_double2(w[q].x / nv, w[q].y / nv) : make_double2(0.0, 0.0);
      TB vb;
      vb.x = v.x;
      vb.y = v.y;
      v = make_double2((double)vb.x, (double)vb.y);
      Vnext[(size_t)s * ldv + r0 + r] = v;
      if ((void*)Vbnext != (void*)Vnext) Vbnext[(size_t)s * ldv + r0 + r] = vb;
    }
  }
  if (c == 0) {
    double2* hq = const_cast<double2*>(ga.h) + (size_t)s * ga.mp2;
    for (int k = tid; k <= j; k += NTH) hq[k] = hs[k];
    if (tid == 0) hq[j + 1] = make_double2(nv, 0.0);
  }
  cl.sync();
}

// V_0 = b / beta rounded to fp32 (the fp32-basis solves): the fp32 copy and its exact fp64 value.
__global__ void round_basis_kernel(double2* __restrict__ V, float2* __restrict__ Vf, int64_t ldv, int64_t n,
                                   uint64_t active, const unsigned long long* __restrict__ dmask) {
  const int s = blockIdx.y;
  if (!sys_on(active, dmask, s)) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 v = V[(size_t)s * ldv + i];
  const float2 f = make_float2((float)v.x, (float)v.y);
  Vf[(size_t)s * ldv + i] = f;
  V[(size_t)s * ldv + i] = make_double2((double)f.x, (double)f.y);
}

// The Givens steps of every active system in parallel (one warp each), after the fused
// Arnoldi step; the sequential rotation chain of one system no longer holds a cluster.
__global__ void __launch_bounds__(32) givens_kernel(uint64_t active, GivensArgs ga, unsigned* done_cnt,
                                                    volatile unsigned long long* publish) {
  extern __shared__ __align__(16) double2 gsm2[];
  const int s = blockIdx.x;
  if (sys_on(active, ga.mask, s)) givens_block(ga, s, gsm2);
  // the last block to finish publishes the convergence mask to the host ring
  __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done_cnt, 1u) == gridDim.x - 1) {
      *done_cnt = 0u;
      __threadfence();
      *publish = *(volatile unsigned long long*)ga.mask;
      __threadfence_system();
    }
  }
}

// Per-thread, per-device host resources: a pinned ring for the convergence mask and
// its events, plus reusable timing events.
struct HostSync {
  unsigned long long* ring = nullptr;      // pinned, host-mapped
  unsigned long long* ring_dev = nullptr;  // its device alias
  cudaEvent_t ev[kRing] = {};
  std::vector<cudaEvent_t> timing[2];
  HostSync() = default;
  HostSync(const HostSync&) = delete;
  HostSync& operator=(const HostSync&) = delete;
  // released when the owning thread exits (worker threads of a sweep come and go);
  // errors at process teardown (context already gone) are ignored
  ~HostSync() {
    if (ring) cudaFreeHost(ring);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& v : timing)
      for (auto& e : v) cudaEventDestroy(e);
    cudaGetLastError();
  }
};

HostSync* host_sync() {
  thread_local std::map<int, HostSync> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  HostSync& h = per_dev[dev];
  if (!h.ring) {
    if (cudaHostAlloc(&h.ring, sizeof(unsigned long long) * kRing, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&h.ring_dev, h.ring, 0) != cudaSuccess) {
      h.ring = nullptr;
      return nullptr;
    }
    for (auto& e : h.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
  }
  return &h;
}

}  // namespace

cudaEvent_t timing_event(int slot, size_t i) {
  HostSync* h = host_sync();
  if (!h) return nullptr;
  auto& v = h->timing[slot];
  while (v.size() <= i) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    v.push_back(e);
  }
  return v[i];
}

size_t krylov_workspace(int nsys, int64_t n, int64_t ldv, int max_iter, Carver& c, KrylovWs* w) {
  const int m = max_iter;
  const int nchunk = (int)((n + kKrylovChunk - 1) / kKrylovChunk);
  KrylovWs t;
  t.V = c.take<double2>((size_t)(m + 1) * nsys * ldv);
  t.W = c.take<double2>((size_t)(m > 0 ? m : 1) * nsys * ldv);
  t.Vf = c.take<float2>((size_t)(m + 1) * nsys * ldv);
  t.w = c.take<double2>((size_t)nsys * ldv);
  t.part = c.take<double2>((size_t)nsys * (m + 1) * nchunk);
  t.h = c.take<double2>((size_t)nsys * (m + 2));
  t.h2 = c.take<double2>((size_t)nsys * (m + 2));
  t.y = c.take<double2>((size_t)nsys * m);
  t.npart = c.take<double2>((size_t)nsys * ((n + kT - 1) / kT));
  t.H = c.take<double2>((size_t)nsys * m * (m + 1));
  t.cs = c.take<double2>((size_t)nsys * m);
  t.sn = c.take<double2>((size_t)nsys * m);
  t.gam = c.take<double2>((size_t)nsys * (m + 1));
  t.sys = c.take<DevSys>(nsys);
  t.mask = c.take<unsigned long long>(1);
  t.cnt = c.take<unsigned>(2 * 64 + 1);  // [128]: the Givens kernel's last-block counter
  if (w) *w = t;
  return c.bytes();
}

nat_status gmres_batched(int nsys, int64_t n, int64_t ldv, const double2* b, double2* x, const KrylovOp& op,
                         double tol, int max_iter, const KrylovWs& ws, std::vector<KrylovResult>& res,
                         cudaStream_t s, double* t_op_s, bool basis32) {
  if (nsys < 1 || nsys > 64) return fail(NAT_ERR_INVALID_ARG, "batched GMRES supports 1..64 systems");
  const int m = max_iter, mp1 = m + 1, mp2 = m + 2;
  const int nchunk = (int)((n + kKrylovChunk - 1) / kKrylovChunk);
  const size_t vstride = (size_t)nsys * ldv;
  const unsigned gx = (unsigned)((n + kT - 1) / kT);
  const uint64_t all = nsys == 64 ? ~0ull : ((1ull << nsys) - 1);
  const size_t gsmem = sizeof(double2) * (mp1 + 2 * (size_t)m);
  if (gsmem > (size_t)kBackSmemMax) return fail(NAT_ERR_INVALID_ARG, "max_iter %d too large", m);
  if (gsmem > 48 * 1024)
    NAT_CUDA_TRY(cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
  HostSync* hs = host_sync();
  if (!hs) return fail(NAT_ERR_CUDA, "pinned host ring / events: %s", cudaGetErrorString(cudaGetLastError()));
  res.assign(nsys, KrylovResult{0, 1, 0.0});

  NAT_CUDA_TRY(cudaMemsetAsync(ws.cnt, 0, sizeof(unsigned) * (2 * 64 + 1), s));
  // dots of nvec basis vectors (or of w with itself) with w, reduced into h / h2
  auto dots = [&](const double2* Vb, size_t vs, const double2* w, int nvec, const unsigned long long* dm, int mode,
                  int slot) {
    dots_kernel<<<dim3(nchunk, nvec, nsys), kT, 0, s>>>(Vb, vs, ldv, w, n, nvec, nchunk, mp1, all, dm, ws.part, mp2,
                                                       mode, slot, ws.h, ws.h2, ws.cnt);
  };
  // beta = ||b||, V0 = b / beta
  dots(b, 0, b, 1, nullptr, 2, 0);
  gm_init_kernel<<<1, 64, 0, s>>>(nsys, mp1, mp2, ws.h, ws.gam, ws.sys, ws.mask);
  scale_kernel<<<dim3(gx, nsys), kT, 0, s>>>(b, ldv, n, mp2, 0, all, ws.mask, ws.h, ws.V, nullptr);
  NAT_LAUNCH_CHECK();

  GivensArgs ga{0, m, mp1, mp2, tol, ws.h, ws.H, ws.cs, ws.sn, ws.gam, ws.sys, ws.mask};
  // fused Arnoldi step (one cluster launch per iteration) for short vectors; NAT_GMRES_FUSED=0
  // selects the multi-kernel path (A/B comparisons)
  static const bool fused_env = [] {
    const char* e = std::getenv("NAT_GMRES_FUSED");
    return !(e && e[0] == '0');
  }();
  // fused-step shape (nat_krylov_config, else NAT_FUSED_CL / NAT_FUSED_NTH / NAT_FUSED_SMEM_KB):
  // CTAs per system 4 (default), 8, or 2 (fp32 basis); 512 threads (2 update groups, leaving
  // registers for pair-kernel CTAs of other streams) or 256 (fp32 basis); the shared-memory
  // residency cap (default 120 KB: one CTA per SM keeps the clusters' basis slices in L2)
  const KrylovConfig kc = krylov_config();
  const int fused_cl = (kc.cl == 2 && !basis32) ? 4 : kc.cl;
  const int64_t rpc = (n + fused_cl - 1) / fused_cl;
  const bool fused = fused_env && n <= (int64_t)fused_cl * kT * kFusedMaxRT;
  const int need_rt = (int)((rpc + kT - 1) / kT);
  const int fused_rt = need_rt <= 1 ? 1 : need_rt <= 2 ? 2 : need_rt <= 4 ? 4 : 8;
  const size_t fused_cap = (size_t)kc.smem_kb * 1024;
  const bool fused_narrow = kc.nth != 768;
  const bool fused_256 = kc.nth == 256;
  const int fused_kg = (basis32 && fused_256 && fused_cl != 8) ? 1 : (fused_cl != 2 && fused_rt <= 2 && !fused_narrow) ? 3 : 2;
  const int fused_nth = fused_kg * kT;
  const size_t fsmem = std::max(fused_cap, sizeof(double2) * ((size_t)rpc * fused_kg + 4 * (size_t)mp1));
  using FusedFn = void (*)(const double2*, size_t, int64_t, int64_t, int64_t, const double2*, double2*, uint64_t,
                           GivensArgs);
  FusedFn fused_fn = nullptr;
  if (fused_cl == 8 && fused_kg == 3)
    fused_fn = fused_rt == 1 ? arnoldi_fused_kernel<1, 768, 8> : arnoldi_fused_kernel<2, 768, 8>;
  else if (fused_cl == 8)  // the kernel's thread count must match the launch (fused_nth)
    fused_fn = fused_rt == 1 ? arnoldi_fused_kernel<1, 512, 8> : fused_rt == 2 ? arnoldi_fused_kernel<2, 512, 8>
             : fused_rt == 4 ? arnoldi_fused_kernel<4, 512, 8> : arnoldi_fused_kernel<8, 512, 8>;
  else if (fused_kg == 3)
    fused_fn = fused_rt == 1 ? arnoldi_fused_kernel<1, 768, 4> : fused_rt == 2 ? arnoldi_fused_kernel<2, 768, 4>
             : fused_rt == 4 ? arnoldi_fused_kernel<4, 512, 4> : arnoldi_fused_kernel<8, 512, 4>;
  else
    fused_fn = fused_rt == 1 ? arnoldi_fused_kernel<1, 512, 4> : fused_rt == 2 ? arnoldi_fused_kernel<2, 512, 4>
             : fused_rt == 4 ? arnoldi_fused_kernel<4, 512, 4> : arnoldi_fused_kernel<8, 512, 4>;
  // fused v2 kernel: always for the fp32 basis; NAT_GMRES_V2 = 1 also for the fp64 basis
  static const bool v2_env = [] {
    const char* e = std::getenv("NAT_GMRES_V2");
    return e && e[0] == '1';
  }();
  const bool b32 = basis32 && fused;
  using FusedV2d = void (*)(const double2*, size_t, int64_t, int64_t, int64_t, const double2*, double2*, double2*,
                            uint64_t, GivensArgs);
  using FusedV2f = void (*)(const float2*, size_t, int64_t, int64_t, int64_t, const double2*, double2*, float2*,
                            uint64_t, GivensArgs);
  FusedV2d v2d = nullptr;
  FusedV2f v2f = nullptr;
  if (fused && fused_cl == 2 && b32) {
    v2f = fused_kg == 1 ? (fused_rt == 2 ? arnoldi_fused_v2_kernel<float2, 2, 256, 2> : fused_rt == 4 ? arnoldi_fused_v2_kernel<float2, 4, 256, 2>
                                                                                   : arnoldi_fused_v2_kernel<float2, 8, 256, 2>)
                        : (fused_rt == 2 ? arnoldi_fused_v2_kernel<float2, 2, 512, 2> : fused_rt == 4 ? arnoldi_fused_v2_kernel<float2, 4, 512, 2>
                                                                                     : arnoldi_fused_v2_kernel<float2, 8, 512, 2>);
    if (fused_rt == 1) v2f = fused_kg == 1 ? arnoldi_fused_v2_kernel<float2, 1, 256, 2> : arnoldi_fused_v2_kernel<float2, 1, 512, 2>;
  } else if (fused && fused_cl == 4 && fused_kg == 1 && b32) {
    v2f = fused_rt == 1 ? arnoldi_fused_v2_kernel<float2, 1, 256, 4> : fused_rt == 2 ? arnoldi_fused_v2_kernel<float2, 2, 256, 4>
        : fused_rt == 4 ? arnoldi_fused_v2_kernel<float2, 4, 256, 4> : arnoldi_fused_v2_kernel<float2, 8, 256, 4>;
  } else if (fused && fused_cl == 4 && fused_kg == 2) {
    if (b32)
      v2f = fused_rt == 1 ? arnoldi_fused_v2_kernel<float2, 1, 512, 4> : fused_rt == 2 ? arnoldi_fused_v2_kernel<float2, 2, 512, 4>
          : fused_rt == 4 ? arnoldi_fused_v2_kernel<float2, 4, 512, 4> : arnoldi_fused_v2_kernel<float2, 8, 512, 4>;
    else if (v2_env)
      v2d = fused_rt == 1 ? arnoldi_fused_v2_kernel<double2, 1, 512, 4> : fused_rt == 2 ? arnoldi_fused_v2_kernel<double2, 2, 512, 4>
          : fused_rt == 4 ? arnoldi_fused_v2_kernel<double2, 4, 512, 4> : arnoldi_fused_v2_kernel<double2, 8, 512, 4>;
  }
  const bool use_b32 = v2f != nullptr;
  if (fused) {
    if (fsmem > (size_t)kBackSmemMax) return fail(NAT_ERR_INVALID_ARG, "max_iter %d too large", m);
    if (v2f) NAT_CUDA_TRY(cudaFuncSetAttribute((const void*)v2f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
    if (v2d) NAT_CUDA_TRY(cudaFuncSetAttribute((const void*)v2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
    if (gsmem > 48 * 1024)
      NAT_CUDA_TRY(cudaFuncSetAttribute(givens_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
    NAT_CUDA_TRY(cudaFuncSetAttribute((const void*)fused_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
  }
  int n_timed = 0;
  auto enqueue = [&](int j, uint64_t host_active) -> nat_status {
    double2* Vj = ws.V + (size_t)j * vstride;
    double2* Wj = ws.W + (size_t)j * vstride;  // A V_j, kept for the final residual
    if (t_op_s) {
      cudaEvent_t e0 = timing_event(0, 2 * j), e1 = timing_event(0, 2 * j + 1);
      if (!e0 || !e1) return fail(NAT_ERR_CUDA, "timing events");
      NAT_CUDA_TRY(cudaEventRecord(e0, s));
      nat_status stt = op(Vj, Wj, host_active, ws.mask, s);
      if (stt != NAT_OK) return stt;
      NAT_CUDA_TRY(cudaEventRecord(e1, s));
      n_timed = j + 1;
    } else {
      nat_status stt = op(Vj, Wj, host_active, ws.mask, s);
      if (stt != NAT_OK) return stt;
    }
    ga.j = j;
    if (fused) {  // short vectors: the whole CGS2 step in one cluster launch per iteration
      const dim3 grid(fused_cl, nsys);
      cudaError_t e = cudaSuccess;
      if (v2f)
        v2f<<<grid, fused_nth, fsmem, s>>>(ws.Vf, vstride, ldv, n, rpc, Wj, ws.V + (size_t)(j + 1) * vstride,
                                           ws.Vf + (size_t)(j + 1) * vstride, all, ga);
      else if (v2d)
        v2d<<<grid, fused_nth, fsmem, s>>>(ws.V, vstride, ldv, n, rpc, Wj, ws.V + (size_t)(j + 1) * vstride,
                                           ws.V + (size_t)(j + 1) * vstride, all, ga);
      else
        fused_fn<<<grid, fused_nth, fsmem, s>>>(ws.V, vstride, ldv, n, rpc, Wj, ws.V + (size_t)(j + 1) * vstride, all, ga);
      e = cudaGetLastError();
      if (e != cudaSuccess) return fail(NAT_ERR_CUDA, "fused Arnoldi launch: %s", cudaGetErrorString(e));
      givens_kernel<<<nsys, 32, gsmem, s>>>(all, ga, ws.cnt + 128, hs->ring_dev + j % kRing);
      NAT_LAUNCH_CHECK();
    } else {
      for (int pass = 0; pass < 2; ++pass) {  // CGS2 (w = W_j minus its projections); pass 1 also forms ||w||
        const double2* win = pass == 0 ? Wj : ws.w;
        dots(ws.V, vstride, win, j + 1, ws.mask, pass, 0);
        update_kernel<<<dim3(gx, nsys), kT, pass == 1 ? gsmem : 0, s>>>(
            ws.V, vstride, ldv, n, j + 1, mp2, all, ws.mask, ws.h2, win, ws.w, pass == 1 ? j + 1 : -1, ws.h,
            ws.npart, ws.cnt + 64, pass == 1, ga);
      }
      scale_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.w, ldv, n, mp2, j + 1, all, ws.mask, ws.h,
                                                 ws.V + (size_t)(j + 1) * vstride, hs->ring_dev + j % kRing);
      NAT_LAUNCH_CHECK();
    }
    NAT_CUDA_TRY(cudaEventRecord(hs->ev[j % kRing], s));
    return NAT_OK;
  };
  // Iteration j is enqueued with the mask read back after iteration j-2; the host then
  // waits for iteration j-1 while the GPU runs iteration j.
  if (use_b32) {  // V_0 rounded to the fp32 basis (R-basis32)
    round_basis_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.V, ws.Vf, ldv, n, all, ws.mask);
    NAT_LAUNCH_CHECK();
  }
  if (m > 0) {
    nat_status stt = enqueue(0, all);
    if (stt != NAT_OK) return stt;
    uint64_t known = all;
    static const bool dbg = std::getenv("NAT_DEBUG_GMRES") != nullptr;
    double t_enq = 0, t_wait = 0;
    int j = 1;
    for (; j < m; ++j) {
      auto c0 = std::chrono::steady_clock::now();
      stt = enqueue(j, known);
      if (stt != NAT_OK) return stt;
      auto c1 = std::chrono::steady_clock::now();
      NAT_CUDA_TRY(cudaEventSynchronize(hs->ev[(j - 1) % kRing]));
      auto c2 = std::chrono::steady_clock::now();
      t_enq += std::chrono::duration<double>(c1 - c0).count();
      t_wait += std::chrono::duration<double>(c2 - c1).count();
      known = *(volatile unsigned long long*)&hs->ring[(j - 1) % kRing];
      if (!known) break;
    }
    if (dbg)
      std::fprintf(stderr, "[gmres] nsys=%d n=%lld iters<=%d host enqueue %.1f us/it, wait %.1f us/it\n", nsys,
                   (long long)n, j, 1e6 * t_enq / j, 1e6 * t_wait / j);
  }
  {
    // the kernel stages the triangle when k(k+1)/2 entries fit next to r and y
    const size_t base = sizeof(double2) * 2 * (size_t)m;
    if (base > (size_t)kBackSmemMax) return fail(NAT_ERR_INVALID_ARG, "max_iter %d too large", m);
    const size_t smem = std::min(base + sizeof(double2) * (size_t)m * (m + 1) / 2, (size_t)kBackSmemMax);
    if (smem > 48 * 1024)
      NAT_CUDA_TRY(cudaFuncSetAttribute(backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    backsolve_kernel<<<nsys, kBackT, smem, s>>>(m, mp1, ws.H, ws.gam, ws.sys, ws.y, (int)smem);
  }
  // x = V y and the true residual b - A x = b - sum_k y_k (A V_k), then ||b - A x|| / beta
  combine_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.V, ws.W, vstride, ldv, n, m, ws.y, ws.sys, b, x, ws.w);
  dots(ws.w, 0, ws.w, 1, nullptr, 2, 0);
  NAT_LAUNCH_CHECK();
  NAT_LAUNCH_CHECK();
  std::vector<double2> hbuf((size_t)nsys * mp2);
  std::vector<DevSys> sys(nsys);
  NAT_CUDA_TRY(cudaMemcpyAsync(hbuf.data(), ws.h, sizeof(double2) * nsys * mp2, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaMemcpyAsync(sys.data(), ws.sys, sizeof(DevSys) * nsys, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < nsys; ++q) {
    if (sys[q].flags & kSysNonFinite) {
      if (sys[q].k == 0) return fail(NAT_ERR_NUMERIC, "non-finite right-hand side (system %d)", q);
      return fail(NAT_ERR_NUMERIC, "non-finite Arnoldi norm (system %d, iteration %d)", q, sys[q].k - 1);
    }
    const double rn = hbuf[(size_t)q * mp2].x;
    if (!std::isfinite(rn)) return fail(NAT_ERR_NUMERIC, "non-finite residual (system %d)", q);
    res[q].iters = sys[q].k;
    res[q].converged = (sys[q].flags & kSysConverged) ? 1 : 0;
    res[q].rel_residual = sys[q].beta > 0 ? rn / sys[q].beta : 0.0;
  }
  if (t_op_s) {
    double t = 0;
    for (int j = 0; j < n_timed; ++j) {
      float ms = 0.f;
      NAT_CUDA_TRY(cudaEventElapsedTime(&ms, timing_event(0, 2 * j), timing_event(0, 2 * j + 1)));
      t += 1e-3 * ms;
    }
    *t_op_s = t;
  }
  return NAT_OK;
}

}  // namespace nat

// ------------------------------------------------------------------------------------
// dense BEM solve, row-sharded
// ------------------------------------------------------------------------------------
namespace {
struct SolveLayout {
  int rank, world;
  int64_t rpr, ldv;
};

SolveLayout layout(nat_comm* comm, int64_t n) {
  SolveLayout L;
  L.rank = comm ? comm->rank : 0;
  L.world = comm ? comm->world : 1;
  L.rpr = (n + L.world - 1) / L.world;
  L.ldv = L.rpr * L.world;  // padded gather length
  return L;
}

size_t solve_ws(nat_comm* comm, int64_t n, int max_iter, nat::Carver& c, nat::KrylovWs* kw, double2** bfull,
                double2** xfull) {
  SolveLayout L = layout(comm, n);
  nat::krylov_workspace(1, n, L.ldv, max_iter, c, kw);
  *bfull = c.take<double2>(L.ldv);
  *xfull = c.take<double2>(L.ldv);
  return c.bytes();
}
}  // namespace

extern "C" size_t nat_bem_solve_workspace(nat_prec prec, int64_t n, int64_t rows_local, int max_iter) {
  (void)prec;
  (void)rows_local;
  if (max_iter <= 0) max_iter = 200;
  nat::Carver c(nullptr);
  nat::KrylovWs kw;
  double2 *bf, *xf;
  // sized for the worst padding (world up to 64)
  int64_t npad = n + 64;
  nat::krylov_workspace(1, n, npad, max_iter, c, &kw);
  c.take<double2>(npad);
  c.take<double2>(npad);
  (void)bf;
  (void)xf;
  return c.bytes();
}

extern "C" nat_status nat_bem_solve(nat_comm* comm, nat_prec prec, int64_t n, int64_t row_begin, int64_t row_end,
                                    const void* A_local, int64_t lda, const void* b_local, void* x, double tol,
                                    int max_iter, void* ws, size_t ws_bytes, nat_solve_info* info,
                                    nat_stream_t stream) {
  NAT_TRACE();
  auto t_start = std::chrono::steady_clock::now();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(n >= 1 && lda >= n, "need n >= 1 and lda >= n");
  if (tol <= 0) tol = 1e-6;
  if (max_iter <= 0) max_iter = 200;
  SolveLayout L = layout(comm, n);
  NAT_REQUIRE(L.world <= 64, "world size %d > 64", L.world);
  // the same condition on every rank (no rank fails alone before a collective)
  NAT_REQUIRE((int64_t)(L.world - 1) * L.rpr < n, "the last of %d ranks owns no rows (n = %lld)", L.world,
              (long long)n);
  const int64_t rb = L.rank * L.rpr, re = nat::min64(n, rb + L.rpr);
  NAT_REQUIRE(row_begin == rb && row_end == re,
              "rank %d must own rows [%lld, %lld) (rows_per_rank = ceil(n/world)); got [%lld, %lld)", L.rank,
              (long long)rb, (long long)re, (long long)row_begin, (long long)row_end);
  NAT_REQUIRE(prec == NAT_FP64 || (lda % 2 == 0 && ((uintptr_t)A_local % 16) == 0),
              "NAT_FP32 needs an even lda and a 16-byte aligned A");
  NAT_REQUIRE_DEV(A_local);
  NAT_REQUIRE_DEV(b_local);
  NAT_REQUIRE_DEV(x);
  NAT_REQUIRE_DEV(ws);
  nat::Carver c(ws);
  nat::KrylovWs kw;
  double2 *bfull, *xfull;
  size_t need = solve_ws(comm, n, max_iter, c, &kw, &bfull, &xfull);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows = row_end - row_begin;
  int n_comm = 0;
  // gather b
  NAT_CUDA_TRY(cudaMemsetAsync(bfull, 0, sizeof(double2) * L.ldv, s));
  NAT_CUDA_TRY(cudaMemcpyAsync(bfull + rb, b_local, sizeof(double2) * rows, cudaMemcpyDeviceToDevice, s));
  if (L.world > 1) {
    nat_status st = nat::allgather_inplace(comm, (double*)bfull, (size_t)L.rpr * 2, s);
    if (st != NAT_OK) return st;
  }
  auto op = [&](const double2* in, double2* out, uint64_t, const unsigned long long* dmask,
                cudaStream_t ss) -> nat_status {
    nat_status st = nat::matvec_internal(prec, rows, n, A_local, lda, in, out + rb, ss, dmask);
    if (st != NAT_OK) return st;
    if (L.world > 1) {  // every rank enqueues the same iterations (replicated, deterministic mask)
      cudaEvent_t e0 = info ? nat::timing_event(1, 2 * n_comm) : nullptr;
      cudaEvent_t e1 = info ? nat::timing_event(1, 2 * n_comm + 1) : nullptr;
      if (e0 && e1) NAT_CUDA_TRY(cudaEventRecord(e0, ss));
      st = nat::allgather_inplace(comm, (double*)out, (size_t)L.rpr * 2, ss);
      if (e0 && e1) {
        NAT_CUDA_TRY(cudaEventRecord(e1, ss));
        ++n_comm;
      }
    }
    return st;
  };
  std::vector<nat::KrylovResult> res;
  double t_op = 0;
  nat_status st = nat::gmres_batched(1, n, L.ldv, bfull, xfull, op, tol, max_iter, kw, res, s,
                                     info ? &t_op : nullptr);
  if (st != NAT_OK) return st;
  NAT_CUDA_TRY(cudaMemcpyAsync(x, xfull, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  double t_comm = 0;
  for (int c = 0; c < n_comm; ++c) {
    float ms = 0.f;
    NAT_CUDA_TRY(cudaEventElapsedTime(&ms, nat::timing_event(1, 2 * c), nat::timing_event(1, 2 * c + 1)));
    t_comm += 1e-3 * ms;
  }
  if (info) {
    info->iters = res[0].iters;
    info->converged = res[0].converged;
    info->rel_residual = res[0].rel_residual;
    info->t_matvec_s = t_op;
    info->t_comm_s = t_comm;
    info->t_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
  return res[0].converged ? NAT_OK : NAT_WARN_NOT_CONVERGED;
}

// ------------------------------------------------------------------------------------
// NEXT-3: the same row-sharded GMRES over the matrix-free operator (nat_bem_mf_*)
// ------------------------------------------------------------------------------------
extern "C" size_t nat_bem_mf_solve_workspace(const nat_bem_mf* op, int max_iter, int world) {
  if (!op || !op->mesh) return 0;
  if (max_iter <= 0) max_iter = 200;
  if (world < 1) world = 1;
  const int64_t n = op->mesh->n_tri;
  const int64_t ldv = (n + world - 1) / world * world;
  nat::Carver c(nullptr);
  nat::krylov_workspace(1, n, ldv, max_iter, c, nullptr);
  c.take<double2>(ldv);
  c.take<double2>(ldv);
  c.take<char>(nat::mf_apply_ws(op));
  return c.bytes();
}

extern "C" nat_status nat_bem_mf_solve(nat_comm* comm, const nat_bem_mf* op, const void* b_local, void* x,
                                       double tol, int max_iter, void* ws, size_t ws_bytes, nat_solve_info* info,
                                       nat_stream_t stream) {
  NAT_TRACE();
  auto t_start = std::chrono::steady_clock::now();
  NAT_REQUIRE(op && op->mesh, "op must be non-null");
  const int64_t n = op->mesh->n_tri;
  if (tol <= 0) tol = 1e-6;
  if (max_iter <= 0) max_iter = 200;
  SolveLayout L = layout(comm, n);
  NAT_REQUIRE(L.world <= 64, "world size %d > 64", L.world);
  NAT_REQUIRE((int64_t)(L.world - 1) * L.rpr < n, "the last of %d ranks owns no rows (n = %lld)", L.world,
              (long long)n);
  const int64_t rb = L.rank * L.rpr, re = nat::min64(n, rb + L.rpr);
  NAT_REQUIRE(op->row_begin == rb && op->row_end == re,
              "rank %d must own rows [%lld, %lld) (rows_per_rank = ceil(n/world)); got [%lld, %lld)", L.rank,
              (long long)rb, (long long)re, (long long)op->row_begin, (long long)op->row_end);
  NAT_REQUIRE_DEV(b_local);
  NAT_REQUIRE_DEV(x);
  NAT_REQUIRE_DEV(ws);
  nat::Carver c(ws);
  nat::KrylovWs kw;
  double2 *bfull, *xfull;
  solve_ws(comm, n, max_iter, c, &kw, &bfull, &xfull);
  const size_t mfb = nat::mf_apply_ws(op);
  void* mfws = c.take<char>(mfb);
  const size_t need = c.bytes();
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  nat_status st = nat::mf_begin(op, mfws, mfb, s);
  if (st != NAT_OK) return st;
  const int64_t rows = re - rb;
  int n_comm = 0;
  NAT_CUDA_TRY(cudaMemsetAsync(bfull, 0, sizeof(double2) * L.ldv, s));
  NAT_CUDA_TRY(cudaMemcpyAsync(bfull + rb, b_local, sizeof(double2) * rows, cudaMemcpyDeviceToDevice, s));
  if (L.world > 1) {
    st = nat::allgather_inplace(comm, (double*)bfull, (size_t)L.rpr * 2, s);
    if (st != NAT_OK) return st;
  }
  auto opf = [&](const double2* in, double2* out, uint64_t, const unsigned long long* dmask,
                 cudaStream_t ss) -> nat_status {
    nat_status stt = nat::mf_apply(op, mfws, in, out + rb, dmask, ss);
    if (stt != NAT_OK) return stt;
    if (L.world > 1) {
      cudaEvent_t e0 = info ? nat::timing_event(1, 2 * n_comm) : nullptr;
      cudaEvent_t e1 = info ? nat::timing_event(1, 2 * n_comm + 1) : nullptr;
      if (e0 && e1) NAT_CUDA_TRY(cudaEventRecord(e0, ss));
      stt = nat::allgather_inplace(comm, (double*)out, (size_t)L.rpr * 2, ss);
      if (e0 && e1) {
        NAT_CUDA_TRY(cudaEventRecord(e1, ss));
        ++n_comm;
      }
    }
    return stt;
  };
  std::vector<nat::KrylovResult> res;
  double t_op = 0;
  st = nat::gmres_batched(1, n, L.ldv, bfull, xfull, opf, tol, max_iter, kw, res, s, info ? &t_op : nullptr);
  if (st != NAT_OK) return st;
  NAT_CUDA_TRY(cudaMemcpyAsync(x, xfull, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  double t_comm = 0;
  for (int q = 0; q < n_comm; ++q) {
    float ms = 0.f;
    NAT_CUDA_TRY(cudaEventElapsedTime(&ms, nat::timing_event(1, 2 * q), nat::timing_event(1, 2 * q + 1)));
    t_comm += 1e-3 * ms;
  }
  if (info) {
    info->iters = res[0].iters;
    info->converged = res[0].converged;
    info->rel_residual = res[0].rel_residual;
    info->t_matvec_s = t_op;
    info->t_comm_s = t_comm;
    info->t_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
  return res[0].converged ? NAT_OK : NAT_WARN_NOT_CONVERGED;
}

extern "C" nat_status nat_krylov_config(int cluster_ctas, int threads, int smem_cap_kb) {
  NAT_REQUIRE(cluster_ctas == 2 || cluster_ctas == 4 || cluster_ctas == 8, "cluster_ctas = %d must be 2, 4 or 8",
              cluster_ctas);
  NAT_REQUIRE(threads == 256 || threads == 512 || threads == 768, "threads = %d must be 256, 512 or 768", threads);
  NAT_REQUIRE(smem_cap_kb >= 0 && smem_cap_kb <= 200, "smem_cap_kb = %d must be in [0, 200]", smem_cap_kb);
  nat::krylov_config();  // settle the environment defaults first
  nat::g_kcfg_cl.store(cluster_ctas);
  nat::g_kcfg_nth.store(threads);
  nat::g_kcfg_smem.store(smem_cap_kb);
  return NAT_OK;
}
