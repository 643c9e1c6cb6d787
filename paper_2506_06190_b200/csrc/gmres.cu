// Row a7 — unrestarted GMRES ("a tolerance of 1e-6 and a maximum of 200
// iterations"; reading R-gmres), batched over systems, plus the
// row-sharded dense-BEM driver nat_bem_solve (matvec -> NCCL all-gather -> replicated
// Arnoldi).  Arnoldi uses classical Gram-Schmidt applied twice (CGS2): two batched
// dot-product launches instead of j+1 dependent ones per iteration.  All reductions
// use fixed chunking (kKrylovChunk) and fixed in-block trees: deterministic, and
// identical on every rank and for every GPU count.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>

#include "krylov.cuh"
#include "nat_comm.cuh"

namespace nat {
namespace {

constexpr int kT = 256;

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

// Fixed-order sum of the nvec x nchunk partials of system s into h / h2:
// mode 0: h = h2 = sum;  mode 1: h2 = sum, h += sum;  mode 2: h[s][slot] = (sqrt(Re sum), 0)
__device__ void finish_sums(const double2* __restrict__ part, int s, int nvec, int nchunk, int mp1, int mp2,
                            int mode, int slot, double2* __restrict__ h, double2* __restrict__ h2) {
  for (int k = threadIdx.x; k < nvec; k += blockDim.x) {
    double2 t = make_double2(0.0, 0.0);
    for (int c = 0; c < nchunk; ++c) {
      const double2 v = __ldcg(&part[((size_t)s * mp1 + k) * nchunk + c]);
      t.x += v.x;
      t.y += v.y;
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
                                                 double2* __restrict__ part, int mp2, int mode, int slot,
                                                 double2* __restrict__ h, double2* __restrict__ h2,
                                                 unsigned* __restrict__ cnt) {
  __shared__ double2 sm[kT / 32];
  __shared__ bool flag;
  const int c = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  if (!((active >> s) & 1ull)) return;
  const double2* v = V + k * vstride_k + (size_t)s * ldv;
  const double2* ww = w + (size_t)s * ldv;
  const int64_t i0 = (int64_t)c * kKrylovChunk, i1 = nat::min64(n, i0 + kKrylovChunk);
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kT) {
    double2 a = v[i], b = ww[i];
    acc.x += a.x * b.x + a.y * b.y;
    acc.y += a.x * b.y - a.y * b.x;
  }
  double2 r = block_reduce(acc, sm);
  if (threadIdx.x == 0) part[((size_t)s * mp1 + k) * nchunk + c] = r;
  if (last_block(&cnt[s], (unsigned)(nchunk * nvec), &flag))
    finish_sums(part, s, nvec, nchunk, mp1, mp2, mode, slot, h, h2);
}

// w[s][i] -= sum_{k < nvec} h2[s][k] V_k[s][i]; with norm_slot >= 0 also
// h[s][norm_slot] = ||w[s]|| (block partials, last block sums them in fixed order).
__global__ void __launch_bounds__(kT) update_kernel(const double2* __restrict__ V, size_t vstride_k, int64_t ldv,
                                                   int64_t n, int nvec, int mp2, uint64_t active,
                                                   const double2* __restrict__ h2, double2* __restrict__ w,
                                                   int norm_slot, double2* __restrict__ h,
                                                   double2* __restrict__ npart, unsigned* __restrict__ cnt) {
  __shared__ double2 sm[kT / 32];
  __shared__ bool flag;
  const int s = blockIdx.y;
  if (!((active >> s) & 1ull)) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double2 o = make_double2(0.0, 0.0);
  if (i < n) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < nvec; ++k) {
      double2 c = h2[(size_t)s * mp2 + k];
      double2 v = V[k * vstride_k + (size_t)s * ldv + i];
      acc.x += c.x * v.x - c.y * v.y;
      acc.y += c.x * v.y + c.y * v.x;
    }
    o = w[(size_t)s * ldv + i];
    o = make_double2(o.x - acc.x, o.y - acc.y);
    w[(size_t)s * ldv + i] = o;
  }
  if (norm_slot < 0) return;
  const double2 r = block_reduce(make_double2(o.x * o.x + o.y * o.y, 0.0), sm);
  if (threadIdx.x == 0) npart[(size_t)s * gridDim.x + blockIdx.x] = r;
  if (last_block(&cnt[s], gridDim.x, &flag) && threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) t += __ldcg(&npart[(size_t)s * gridDim.x + b]).x;
    h[(size_t)s * mp2 + norm_slot] = make_double2(sqrt(t), 0.0);
  }
}

// dst[s][i] = src[s][i] / h[s][slot]   (slot = norm); zero if the norm is 0
__global__ void scale_kernel(const double2* __restrict__ src, int64_t ldv, int64_t n, int mp2, int slot,
                             uint64_t active, const double2* __restrict__ h, double2* __restrict__ dst) {
  const int s = blockIdx.y;
  if (!((active >> s) & 1ull)) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double nv = h[(size_t)s * mp2 + slot].x;
  double2 v = src[(size_t)s * ldv + i];
  dst[(size_t)s * ldv + i] = nv > 0 ? make_double2(v.x / nv, v.y / nv) : make_double2(0.0, 0.0);
}

// x[s][i] = sum_{k < kmax} y[s][k] V_k[s][i]
__global__ void combine_kernel(const double2* __restrict__ V, size_t vstride_k, int64_t ldv, int64_t n,
                               int kmax, int m, const double2* __restrict__ y, double2* __restrict__ x) {
  const int s = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int k = 0; k < kmax; ++k) {
    double2 c = y[(size_t)s * m + k];
    double2 v = V[k * vstride_k + (size_t)s * ldv + i];
    acc.x += c.x * v.x - c.y * v.y;
    acc.y += c.x * v.y + c.y * v.x;
  }
  x[(size_t)s * ldv + i] = acc;
}

__global__ void sub_kernel(const double2* __restrict__ b, int64_t ldv, int64_t n, double2* __restrict__ w) {
  const int s = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 a = b[(size_t)s * ldv + i], c = w[(size_t)s * ldv + i];
  w[(size_t)s * ldv + i] = make_double2(a.x - c.x, a.y - c.y);
}

using cplx = std::complex<double>;

struct SysState {
  std::vector<cplx> H, cs, sn, gam;  // H column-major (m+1) x m
  double beta = 0;
  int k = 0;
  bool done = false, converged = false;
};

}  // namespace

size_t krylov_workspace(int nsys, int64_t n, int64_t ldv, int max_iter, Carver& c, KrylovWs* w) {
  const int m = max_iter;
  const int nchunk = (int)((n + kKrylovChunk - 1) / kKrylovChunk);
  KrylovWs t;
  t.V = c.take<double2>((size_t)(m + 1) * nsys * ldv);
  t.w = c.take<double2>((size_t)nsys * ldv);
  t.part = c.take<double2>((size_t)nsys * (m + 1) * nchunk);
  t.h = c.take<double2>((size_t)nsys * (m + 2));
  t.h2 = c.take<double2>((size_t)nsys * (m + 2));
  t.y = c.take<double2>((size_t)nsys * m);
  t.npart = c.take<double2>((size_t)nsys * ((n + kT - 1) / kT));
  t.cnt = c.take<unsigned>(2 * 64);
  if (w) *w = t;
  return c.bytes();
}

nat_status gmres_batched(int nsys, int64_t n, int64_t ldv, const double2* b, double2* x, const KrylovOp& op,
                         double tol, int max_iter, const KrylovWs& ws, std::vector<KrylovResult>& res,
                         cudaStream_t s, double* t_op_s) {
  if (nsys < 1 || nsys > 64) return fail(NAT_ERR_INVALID_ARG, "batched GMRES supports 1..64 systems");
  const int m = max_iter, mp1 = m + 1, mp2 = m + 2;
  const int nchunk = (int)((n + kKrylovChunk - 1) / kKrylovChunk);
  const size_t vstride = (size_t)nsys * ldv;
  const unsigned gx = (unsigned)((n + kT - 1) / kT);
  const uint64_t all = nsys == 64 ? ~0ull : ((1ull << nsys) - 1);
  double t_op = 0;  // device time of the operator (CUDA events), if requested
  struct Events {
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } evs;
  cudaEvent_t* ev = evs.e;
  if (t_op_s) {
    NAT_CUDA_TRY(cudaEventCreate(&ev[0]));
    NAT_CUDA_TRY(cudaEventCreate(&ev[1]));
  }
  res.assign(nsys, KrylovResult{0, 1, 0.0});
  std::vector<SysState> st(nsys);
  std::vector<double2> hbuf((size_t)nsys * mp2);

  NAT_CUDA_TRY(cudaMemsetAsync(ws.cnt, 0, sizeof(unsigned) * 2 * 64, s));
  // dots of nvec basis vectors (or of w with itself) with w, reduced into h / h2
  auto dots = [&](const double2* Vb, size_t vs, const double2* w, int nvec, uint64_t act, int mode, int slot) {
    dots_kernel<<<dim3(nchunk, nvec, nsys), kT, 0, s>>>(Vb, vs, ldv, w, n, nvec, nchunk, mp1, act, ws.part, mp2,
                                                       mode, slot, ws.h, ws.h2, ws.cnt);
  };
  // beta = ||b||, V0 = b / beta
  dots(b, 0, b, 1, all, 2, 0);
  NAT_LAUNCH_CHECK();
  NAT_CUDA_TRY(cudaMemcpyAsync(hbuf.data(), ws.h, sizeof(double2) * nsys * mp2, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  uint64_t active = 0;
  for (int q = 0; q < nsys; ++q) {
    double beta = hbuf[(size_t)q * mp2].x;
    if (!std::isfinite(beta)) return fail(NAT_ERR_NUMERIC, "non-finite right-hand side (system %d)", q);
    st[q].beta = beta;
    st[q].H.assign((size_t)mp1 * m, 0.0);
    st[q].cs.assign(m, 0.0);
    st[q].sn.assign(m, 0.0);
    st[q].gam.assign(mp1, 0.0);
    st[q].gam[0] = beta;
    if (beta == 0.0) {
      st[q].done = st[q].converged = true;
    } else {
      active |= 1ull << q;
    }
  }
  scale_kernel<<<dim3(gx, nsys), kT, 0, s>>>(b, ldv, n, mp2, 0, active, ws.h, ws.V);
  NAT_LAUNCH_CHECK();

  for (int j = 0; j < m && active; ++j) {
    double2* Vj = ws.V + (size_t)j * vstride;
    if (t_op_s) NAT_CUDA_TRY(cudaEventRecord(ev[0], s));
    nat_status stt = op(Vj, ws.w, active, s);
    if (stt != NAT_OK) return stt;
    if (t_op_s) NAT_CUDA_TRY(cudaEventRecord(ev[1], s));
    for (int pass = 0; pass < 2; ++pass) {  // CGS2; the second update also forms ||w||
      dots(ws.V, vstride, ws.w, j + 1, active, pass, 0);
      update_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.V, vstride, ldv, n, j + 1, mp2, active, ws.h2, ws.w,
                                                  pass == 1 ? j + 1 : -1, ws.h, ws.npart, ws.cnt + 64);
    }
    scale_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.w, ldv, n, mp2, j + 1, active, ws.h,
                                               ws.V + (size_t)(j + 1) * vstride);
    NAT_LAUNCH_CHECK();
    NAT_CUDA_TRY(cudaMemcpy2DAsync(hbuf.data(), sizeof(double2) * mp2, ws.h, sizeof(double2) * mp2,
                                   sizeof(double2) * (j + 2), nsys, cudaMemcpyDeviceToHost, s));
    NAT_CUDA_TRY(cudaStreamSynchronize(s));
    if (t_op_s) {
      float ms = 0.f;
      NAT_CUDA_TRY(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      t_op += 1e-3 * ms;
    }
    for (int q = 0; q < nsys; ++q) {
      if (!((active >> q) & 1ull)) continue;
      SysState& S = st[q];
      cplx* col = &S.H[(size_t)j * mp1];
      for (int i = 0; i <= j + 1; ++i) col[i] = cplx(hbuf[(size_t)q * mp2 + i].x, hbuf[(size_t)q * mp2 + i].y);
      if (!std::isfinite(col[j + 1].real()))
        return fail(NAT_ERR_NUMERIC, "non-finite Arnoldi norm (system %d, iteration %d)", q, j);
      const bool breakdown = col[j + 1] == 0.0;
      for (int i = 0; i < j; ++i) {
        cplx hi = col[i], hi1 = col[i + 1];
        col[i] = std::conj(S.cs[i]) * hi + std::conj(S.sn[i]) * hi1;
        col[i + 1] = -S.sn[i] * hi + S.cs[i] * hi1;
      }
      cplx a = col[j], bb = col[j + 1];
      double den = std::sqrt(std::norm(a) + std::norm(bb));
      if (den != 0) {
        S.cs[j] = a / den;
        S.sn[j] = bb / den;
      } else {
        S.cs[j] = 1.0;
        S.sn[j] = 0.0;
      }
      col[j] = std::conj(S.cs[j]) * a + std::conj(S.sn[j]) * bb;
      col[j + 1] = 0.0;
      S.gam[j + 1] = -S.sn[j] * S.gam[j];
      S.gam[j] = std::conj(S.cs[j]) * S.gam[j];
      S.k = j + 1;
      if (std::abs(S.gam[j + 1]) <= tol * S.beta || breakdown) {
        S.done = S.converged = true;
        active &= ~(1ull << q);
      } else if (j + 1 == m) {
        S.done = true;
        active &= ~(1ull << q);
      }
    }
  }
  // back-substitution on the host, x = V y on the device
  std::vector<double2> yh((size_t)nsys * m, make_double2(0.0, 0.0));
  int kmax = 0;
  for (int q = 0; q < nsys; ++q) {
    SysState& S = st[q];
    int k = S.k;
    kmax = std::max(kmax, k);
    std::vector<cplx> yy(k);
    for (int i = k - 1; i >= 0; --i) {
      cplx acc = S.gam[i];
      for (int l = i + 1; l < k; ++l) acc -= S.H[(size_t)l * mp1 + i] * yy[l];
      yy[i] = acc / S.H[(size_t)i * mp1 + i];
    }
    for (int i = 0; i < k; ++i) yh[(size_t)q * m + i] = make_double2(yy[i].real(), yy[i].imag());
  }
  if (m > 0)
    NAT_CUDA_TRY(cudaMemcpyAsync(ws.y, yh.data(), sizeof(double2) * nsys * m, cudaMemcpyHostToDevice, s));
  combine_kernel<<<dim3(gx, nsys), kT, 0, s>>>(ws.V, vstride, ldv, n, kmax, m, ws.y, x);
  NAT_LAUNCH_CHECK();
  // true residual ||b - A x|| / beta
  nat_status stt = op(x, ws.w, all, s);
  if (stt != NAT_OK) return stt;
  sub_kernel<<<dim3(gx, nsys), kT, 0, s>>>(b, ldv, n, ws.w);
  dots(ws.w, 0, ws.w, 1, all, 2, 0);
  NAT_LAUNCH_CHECK();
  NAT_CUDA_TRY(cudaMemcpyAsync(hbuf.data(), ws.h, sizeof(double2) * nsys * mp2, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  for (int q = 0; q < nsys; ++q) {
    double rn = hbuf[(size_t)q * mp2].x;
    if (!std::isfinite(rn)) return fail(NAT_ERR_NUMERIC, "non-finite residual (system %d)", q);
    res[q].iters = st[q].k;
    res[q].converged = st[q].converged ? 1 : 0;
    res[q].rel_residual = st[q].beta > 0 ? rn / st[q].beta : 0.0;
  }
  if (t_op_s) *t_op_s = t_op;
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
  auto t_start = std::chrono::steady_clock::now();
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(n >= 1 && lda >= n, "need n >= 1 and lda >= n");
  if (tol <= 0) tol = 1e-6;
  if (max_iter <= 0) max_iter = 200;
  SolveLayout L = layout(comm, n);
  NAT_REQUIRE(L.world <= 64, "world size %d > 64", L.world);
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
  double t_comm = 0;
  // gather b
  NAT_CUDA_TRY(cudaMemsetAsync(bfull, 0, sizeof(double2) * L.ldv, s));
  NAT_CUDA_TRY(cudaMemcpyAsync(bfull + rb, b_local, sizeof(double2) * rows, cudaMemcpyDeviceToDevice, s));
  if (L.world > 1) {
    nat_status st = nat::allgather_inplace(comm, (double*)bfull, (size_t)L.rpr * 2, s);
    if (st != NAT_OK) return st;
  }
  auto op = [&](const double2* in, double2* out, uint64_t, cudaStream_t ss) -> nat_status {
    nat_status st = nat::matvec_internal(prec, rows, n, A_local, lda, in, out + rb, ss);
    if (st != NAT_OK) return st;
    if (L.world > 1) {
      auto t0 = std::chrono::steady_clock::now();
      st = nat::allgather_inplace(comm, (double*)out, (size_t)L.rpr * 2, ss);
      t_comm += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
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
