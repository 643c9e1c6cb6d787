// Row a11 — radiation of the surface field to listener points (reading R-ext):
//   p_m(x_l) = sum_s w_s [ p_ms dG_m/dn_y(x_l, y_s) - g_ms G_m(x_l, y_s) ].
//
// B200 design:
//  * stage kernel folds w/(4 pi) and k into per-source constants (O(S) work):
//      alpha = w p/(4pi), beta = w g/(4pi);  A1 = -Re a, A2 = -k Im a, A3 = k Re a,
//      A4 = -Im a, B1 = -Re b, B2 = -Im b, so that per pair (rho = 1/r, q = (d.n) rho^2)
//      C = q (rho A1 + A2) + rho B1 + i [q (rho A4 + A3) + rho B2],  acc += e^{ikr} C;
//  * main kernel: CTA = 256 threads x R targets each (registers); source tiles of
//    128 records are streamed into shared memory with TMA bulk copies (cp.async.bulk +
//    mbarrier, double buffered) and read back as warp-broadcast LDS.128; MB wavenumbers
//    share r, 1/r and d.n; fp32 math with MUFU rsqrt/sin/cos; a CTA sums its source
//    chunk (<= 8 tiles = 1024 sources) in fp32 registers and writes one fp64 partial;
//  * split-K over source chunks when the target grid is too small for 148 SMs, with a
//    fixed-order fp64 reduction (deterministic, no atomics).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "async_copy.cuh"
#include "nat_internal.cuh"
#include "f32x2.cuh"
#include "pair.cuh"
#include "radiate.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 128;  // sources per shared-memory tile (fp32)
constexpr int kTile64 = 64; // sources per tile (fp64)
constexpr int kMaxChunkTiles = 8;  // fp32 kernel: sources summed in fp32 <= 8 x 128 = 1024, then flushed

template <int MB>
struct Rec {
  static constexpr int NF = ((6 + 6 * MB) + 3) / 4 * 4;  // floats per source record
};

constexpr int kMaxModes = 64;  // wavenumbers per launch (passed by value)
struct KVals {
  float f[kMaxModes];
  double d[kMaxModes];
};

// Kernel kinds: 0 = radiation (G and dG/dn_y, no self exclusion), 1 = MC operator
// (double layer only, self/close pairs excluded), 2 = MC right-hand side (single layer
// only, self/close pairs excluded).  Record per source (each float duplicated for the
// FP32x2 pipe): kind 0: x y z nx ny nz | A1 A2 A3 A4 B1 B2 per mode;  kind 1: x y z nx ny nz |
// A1 A2 A3 A4;  kind 2: x y z | B1 B2.  Padded to a multiple of 4 floats (16-byte loads).
__host__ __device__ constexpr int rec_geo(int kind) { return kind == 2 ? 3 : 6; }
__host__ __device__ constexpr int rec_per_mode(int kind) { return kind == 0 ? 6 : kind == 1 ? 4 : 2; }
__host__ __device__ constexpr int rec_nf(int kind, int MB) {  // floats per record, padded to 16 B
  return ((rec_geo(kind) + rec_per_mode(kind) * MB) + 3) / 4 * 4;
}

struct RadParams {
  const void* rec;      // [n_mchunk][n_src_pad][NF] records
  int64_t n_src_pad;    // multiple of the tile
  int n_tiles;          // n_src_pad / tile
  int chunk_tiles;      // tiles per split
  const double* lis;    // [3][n_lis]
  int64_t n_lis;
  double cx, cy, cz;    // coordinate origin
  KVals k;              // wavenumbers of this launch (<= kMaxModes)
  double2* out;         // [n_split][n_modes][n_lis]
  int n_modes;
  float self_r2;        // SELF mode threshold (see radiate.cuh)
  const unsigned long long* skip;  // see RadInput::skip
  int sub;              // fp32: CTAs per source tile (split s takes sources [s % sub] of tile s / sub)
};

// ------------------------------------------------------------------------------------
// staging
// ------------------------------------------------------------------------------------
// DUP: every value is written twice (x x y y ...), the layout of the FP32x2 kernel.
template <typename T, bool DUP>
struct RecWriter {
  T* r;
  __device__ __forceinline__ void put(int f, double v) const {
    if (DUP) {
      r[2 * f] = (T)v;
      r[2 * f + 1] = (T)v;
    } else {
      r[f] = (T)v;
    }
  }
};

// One CTA stages kStageSrc consecutive sources: each thread builds its record in shared
// memory, then the CTA writes the contiguous block with coalesced 16-byte stores.
constexpr int kStageSrc = 128;
constexpr int kStageMaxBytes = 64 * 4;  // per source: <= 64 floats (fp32) or 32 doubles

template <typename T, bool DUP = false, int SGN = 1>
__global__ void __launch_bounds__(kStageSrc) stage_kernel(int64_t n_src, int64_t n_src_pad, int NF, int MB,
                                                         int n_mchunk, int kind,
                             const double* __restrict__ xyz, const double* __restrict__ nrm,
                             const double* __restrict__ w, double w_const,
                             const double2* __restrict__ p, const double2* __restrict__ g,
                             int64_t ldpg, const KVals kv, int n_modes, double cx,
                             double cy, double cz, T* __restrict__ rec,
                             const unsigned long long* __restrict__ skip) {
  if (skip && *skip == 0ull) return;
  __shared__ __align__(16) unsigned char sbuf[kStageSrc * kStageMaxBytes];
  T* sm = reinterpret_cast<T*>(sbuf);
  const int64_t s0 = (int64_t)blockIdx.x * kStageSrc;
  const int64_t s = s0 + threadIdx.x;
  const int nblk = (int)nat::min64(kStageSrc, n_src_pad - s0);
  double x, y, z, nx, ny, nz, ws;
  if (s < n_src) {
    x = xyz[s] - cx;
    y = xyz[n_src + s] - cy;
    z = xyz[2 * n_src + s] - cz;
    nx = nrm[s];
    ny = nrm[n_src + s];
    nz = nrm[2 * n_src + s];
    ws = (w ? w[s] : w_const) * nat::kInv4Pi;
  } else {  // padding: far away, zero weight -> contributes exactly 0
    x = y = z = 3.0e3;
    nx = 1.0;
    ny = nz = 0.0;
    ws = 0.0;
  }
  // one mode chunk per blockIdx.y (MC shapes: 16 source blocks x up to 64 chunks)
  for (int c = blockIdx.y; c < n_mchunk; c += gridDim.y) {
    if (threadIdx.x < nblk) {
      T* r = sm + (size_t)threadIdx.x * NF;
      const RecWriter<T, DUP> wr{r};
      wr.put(0, x);
      wr.put(1, y);
      wr.put(2, z);
      if (kind != 2) {
        wr.put(3, nx);
        wr.put(4, ny);
        wr.put(5, nz);
      }
      const int G = rec_geo(kind), F = rec_per_mode(kind);
      for (int m = 0; m < MB; ++m) {
        int mode = c * MB + m;
        double ar = 0, ai = 0, br = 0, bi = 0, k = 0;
        if (mode < n_modes && ws != 0.0) {
          double2 pv = p ? p[(size_t)mode * ldpg + s] : make_double2(0.0, 0.0);
          double2 gv = g ? g[(size_t)mode * ldpg + s] : make_double2(0.0, 0.0);
          ar = ws * pv.x;
          ai = ws * pv.y;
          br = ws * gv.x;
          bi = ws * gv.y;
          k = kv.d[mode];
        }
        const int q = G + F * m;
        if (kind != 2) {  // fp32 records (SGN = -1): the kernel forms -d.n (see the main kernel)
          wr.put(q + 0, SGN * -ar);
          wr.put(q + 1, SGN * -k * ai);
          wr.put(q + 2, SGN * k * ar);
          wr.put(q + 3, SGN * -ai);
        }
        if (kind == 0) {
          wr.put(q + 4, -br);
          wr.put(q + 5, -bi);
        } else if (kind == 2) {
          wr.put(q + 0, -br);
          wr.put(q + 1, -bi);
        }
      }
      for (int f = (DUP ? 2 : 1) * (G + F * MB); f < NF; ++f) r[f] = (T)0;
    }
    __syncthreads();
    // NF * sizeof(T) is a multiple of 16 bytes (rec_nf pads to 4 floats; fp64 NF = 12)
    const float4* src4 = reinterpret_cast<const float4*>(sm);
    float4* dst4 = reinterpret_cast<float4*>(rec + ((size_t)c * n_src_pad + s0) * NF);
    const int nvec = (int)((size_t)nblk * NF * sizeof(T) / 16);
    for (int v = threadIdx.x; v < nvec; v += kStageSrc) dst4[v] = src4[v];
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// fp32 main kernel
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------------------------------
// fp32 main kernel on the packed FP32x2 pipe (FADD2 / FMUL2 / FFMA2, sm_100a).
// Two targets share every instruction; each source record is stored duplicated
// (x x y y z z nx nx ...) so a packed operand is one half of an LDS.128 broadcast.
// Per pair: 12.5 FP32-pipe instructions + 3 MUFU (rsqrt, sin, cos) instead of 24 + 3.
// ------------------------------------------------------------------------------------
template <int MB, int KIND>
struct Rec2 {
  static constexpr int NF = rec_nf(KIND, MB);
};

// KIND 1, 2 (SELF): targets coincide with the sources (MC operators): pairs with fp32
// r^2 <= self_r2 (the self pair, d = 0 exactly, and the close pairs evaluated in fp64 by
// the caller) get 1/r = 0, i.e. contribute exactly 0.  NT = threads per CTA (256, or 128
// for fine grids).
template <int R, int MB, int KIND, int NT>
__global__ void __launch_bounds__(NT) radiate_f32x2_kernel(RadParams prm) {
  static_assert(R % 2 == 0, "targets are processed in pairs");
  constexpr int RP = R / 2;
  constexpr bool SELF = KIND != 0;
  constexpr int NF = Rec2<MB, KIND>::NF;
  constexpr int G = rec_geo(KIND), F = rec_per_mode(KIND);
  // short bodies keep cos/sin products in four accumulators (no negation per pair)
  constexpr bool ACC4 = RP * MB <= 2;
  constexpr int kTileFloats = kTile * NF;
  extern __shared__ __align__(128) unsigned char smem[];
  float* buf = reinterpret_cast<float*>(smem);
  __shared__ __align__(8) uint64_t bars[2];
  if (prm.skip && *prm.skip == 0ull) return;

  const int tid = threadIdx.x;
  const int64_t tbase = (int64_t)blockIdx.x * (R * NT);
  const int split = blockIdx.y;
  const int mch = blockIdx.z;

  f2r tx[RP], ty[RP], tz[RP];
#pragma unroll
  for (int p = 0; p < RP; ++p) {
    float c[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t l = tbase + (2 * p + h) * NT + tid;
      if (l >= prm.n_lis) l = prm.n_lis - 1;
      c[h][0] = (float)(prm.lis[l] - prm.cx);
      c[h][1] = (float)(prm.lis[prm.n_lis + l] - prm.cy);
      c[h][2] = (float)(prm.lis[2 * prm.n_lis + l] - prm.cz);
    }
    tx[p] = f2pack(c[0][0], c[1][0]);
    ty[p] = f2pack(c[0][1], c[1][1]);
    tz[p] = f2pack(c[0][2], c[1][2]);
  }
  f2r kk[MB];
#pragma unroll
  for (int m = 0; m < MB; ++m) {
    const float k = prm.k.f[mch * MB + m];
    kk[m] = f2pack(k, k);
  }
  const f2r minus1 = f2pack(-1.f, -1.f);
  // fp32 sums over at most kMaxChunkTiles tiles (1024 sources, the fp32 budget of SURVEY
  // §8(c-8)); split-K partials are then summed in fp64
  f2r ar[RP][MB], ai[RP][MB], br[RP][MB], bi[RP][MB];  // br / bi: ACC4 only
#pragma unroll
  for (int p = 0; p < RP; ++p)
#pragma unroll
    for (int m = 0; m < MB; ++m) ar[p][m] = ai[p][m] = br[p][m] = bi[p][m] = 0ull;
  // fp32 sums flushed to the fp64 output every kMaxChunkTiles tiles (<= 1024 sources in
  // fp32); later flushes of a chunk longer than that add to the output the
  // CTA itself wrote (fixed order, no other CTA touches it)
  auto flush = [&](bool add) {
#pragma unroll
    for (int p = 0; p < RP; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t l = tbase + (2 * p + h) * NT + tid;
        if (l >= prm.n_lis) continue;
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          const int mode = mch * MB + m;
          if (mode >= prm.n_modes) continue;
          double re, im;
          if constexpr (ACC4) {
            re = h ? (double)f2hi(ar[p][m]) - (double)f2hi(br[p][m]) : (double)f2lo(ar[p][m]) - (double)f2lo(br[p][m]);
            im = h ? (double)f2hi(ai[p][m]) + (double)f2hi(bi[p][m]) : (double)f2lo(ai[p][m]) + (double)f2lo(bi[p][m]);
          } else {
            re = h ? (double)f2hi(ar[p][m]) : (double)f2lo(ar[p][m]);
            im = h ? (double)f2hi(ai[p][m]) : (double)f2lo(ai[p][m]);
          }
          double2* o = prm.out + ((size_t)split * prm.n_modes + mode) * prm.n_lis + l;
          if (add) {
            const double2 v = *o;
            re += v.x;
            im += v.y;
          }
          *o = make_double2(re, im);
        }
      }
#pragma unroll
    for (int p = 0; p < RP; ++p)
#pragma unroll
      for (int m = 0; m < MB; ++m) ar[p][m] = ai[p][m] = br[p][m] = bi[p][m] = 0ull;
  };

  // a split is chunk_tiles source tiles, or (sub > 1, one tile per split) a 1/sub part of one
  const int sub = prm.sub;
  const int t0 = (split / sub) * prm.chunk_tiles;
  const int t1 = min(t0 + prm.chunk_tiles, prm.n_tiles);
  const int s_lo = (split % sub) * (kTile / sub), s_hi = s_lo + kTile / sub;
  const float* src = static_cast<const float*>(prm.rec) + (size_t)mch * prm.n_src_pad * NF;
  constexpr uint32_t kBytes = kTileFloats * sizeof(float);

  if (tid == 0) {
    nat::mbar_init(&bars[0], 1);
    nat::mbar_init(&bars[1], 1);
    nat::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int st = 0; st < 2 && t0 + st < t1; ++st) {
      nat::mbar_arrive_expect_tx(&bars[st], kBytes);
      nat::bulk_g2s(buf + st * kTileFloats, src + (size_t)(t0 + st) * kTileFloats, kBytes, &bars[st]);
    }
  }

  for (int it = 0; t0 + it < t1; ++it) {
    const int st = it & 1;
    nat::mbar_wait(&bars[st], (it >> 1) & 1);
    const float4* b4 = reinterpret_cast<const float4*>(buf + st * kTileFloats);

    // short bodies (one target pair, one wavenumber) need a deeper unroll so the
    // shared-memory loads of later sources overlap the arithmetic (ncu r01: LDS-wait)
#ifndef NAT_RAD_UNROLL
#define NAT_RAD_UNROLL 2
#endif
    constexpr int kUnroll = (RP * MB <= 1) ? 4 : NAT_RAD_UNROLL;
#pragma unroll kUnroll
    for (int s = s_lo; s < s_hi; ++s) {
      // one scalar per record field (LDS.128 broadcast), used as the .F32 operand of the
      // packed instructions (both targets of the pair share it)
      float fs[NF];
#pragma unroll
      for (int q = 0; q < NF / 4; ++q) {
        const float4 v = b4[s * (NF / 4) + q];
        fs[4 * q] = v.x;
        fs[4 * q + 1] = v.y;
        fs[4 * q + 2] = v.z;
        fs[4 * q + 3] = v.w;
      }
      auto B = [&](int i) { return f2pack(fs[i], fs[i]); };
#pragma unroll
      for (int p = 0; p < RP; ++p) {
        // e = x - y = -d (the record is the broadcast operand); the staged A coefficients
        // carry the matching sign (d.n = -e.n)
        const f2r dx = f2sub(tx[p], B(0));
        const f2r dy = f2sub(ty[p], B(1));
        const f2r dz = f2sub(tz[p], B(2));
        const f2r r2 = f2fma(dz, dz, f2fma(dy, dy, f2mul(dx, dx)));
        const float r2a = f2lo(r2), r2b = f2hi(r2);
        const float ra = SELF ? (r2a > prm.self_r2 ? rsqrt_approx(r2a) : 0.f) : rsqrt_approx(r2a);
        const float rb = SELF ? (r2b > prm.self_r2 ? rsqrt_approx(r2b) : 0.f) : rsqrt_approx(r2b);
        const f2r rho = f2pack(ra, rb);
        f2r qq = 0ull;
        if constexpr (KIND != 2) {
          const f2r dn = f2fma(dz, B(5), f2fma(dy, B(4), f2mul(dx, B(3))));  // = -d.n
          qq = f2mul(dn, f2mul(rho, rho));
        }
        const f2r rr = f2mul(r2, rho);
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          const f2r kr = f2mul(rr, kk[m]);
          float sa, ca, sb, cb;
          __sincosf(f2lo(kr), &sa, &ca);
          __sincosf(f2hi(kr), &sb, &cb);
          const f2r sn = f2pack(sa, sb), cs = f2pack(ca, cb);
          const int c = G + F * m;  // kind 0: -A1 -A2 -A3 -A4 B1 B2; 1: -A1..-A4; 2: B1 B2
          f2r cr, ci;
          if constexpr (KIND == 0) {
            cr = f2fma(qq, f2fma(rho, B(c), B(c + 1)), f2mul(rho, B(c + 4)));
            ci = f2fma(qq, f2fma(rho, B(c + 3), B(c + 2)), f2mul(rho, B(c + 5)));
          } else if constexpr (KIND == 1) {
            cr = f2mul(qq, f2fma(rho, B(c), B(c + 1)));
            ci = f2mul(qq, f2fma(rho, B(c + 3), B(c + 2)));
          } else {
            cr = f2mul(rho, B(c));
            ci = f2mul(rho, B(c + 1));
          }
          if constexpr (ACC4) {  // (ar - br) + i (ai + bi)
            ar[p][m] = f2fma(cs, cr, ar[p][m]);
            br[p][m] = f2fma(sn, ci, br[p][m]);
            ai[p][m] = f2fma(sn, cr, ai[p][m]);
            bi[p][m] = f2fma(cs, ci, bi[p][m]);
          } else {
            const f2r nci = f2mul(ci, minus1);
            ar[p][m] = f2fma(cs, cr, f2fma(sn, nci, ar[p][m]));
            ai[p][m] = f2fma(sn, cr, f2fma(cs, ci, ai[p][m]));
          }
        }
      }
    }
    if ((it + 1) % kMaxChunkTiles == 0) flush(it + 1 > kMaxChunkTiles);
    __syncthreads();  // every thread is done with buf[st]
    if (tid == 0 && t0 + it + 2 < t1) {
      nat::fence_proxy_async_smem();
      nat::mbar_arrive_expect_tx(&bars[st], kBytes);
      nat::bulk_g2s(buf + st * kTileFloats, src + (size_t)(t0 + it + 2) * kTileFloats, kBytes, &bars[st]);
    }
  }

  if (((t1 - t0) % kMaxChunkTiles) != 0 || t1 == t0) flush(t1 - t0 > kMaxChunkTiles);
}

// ------------------------------------------------------------------------------------
// fp64 main kernel: one wavenumber per pass (MB = 1), R targets per thread, fp64 math.
// ------------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(kThreads) radiate_f64_kernel(RadParams prm) {
  constexpr int NF = 12;
  constexpr int kTileD = kTile64 * NF;
  extern __shared__ __align__(128) unsigned char smem[];
  double* buf = reinterpret_cast<double*>(smem);
  __shared__ __align__(8) uint64_t bars[2];
  if (prm.skip && *prm.skip == 0ull) return;
  const int tid = threadIdx.x;
  const int64_t tbase = (int64_t)blockIdx.x * (R * kThreads);
  const int split = blockIdx.y, mch = blockIdx.z;
  double tx[R], ty[R], tz[R], ar[R], ai[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t l = tbase + r * kThreads + tid;
    if (l >= prm.n_lis) l = prm.n_lis - 1;
    tx[r] = prm.lis[l] - prm.cx;
    ty[r] = prm.lis[prm.n_lis + l] - prm.cy;
    tz[r] = prm.lis[2 * prm.n_lis + l] - prm.cz;
    ar[r] = ai[r] = 0.0;
  }
  const double k = prm.k.d[mch];
  const int t0 = split * prm.chunk_tiles;
  const int t1 = min(t0 + prm.chunk_tiles, prm.n_tiles);
  const double* src = static_cast<const double*>(prm.rec) + (size_t)mch * prm.n_src_pad * NF;
  constexpr uint32_t kBytes = kTileD * sizeof(double);
  if (tid == 0) {
    nat::mbar_init(&bars[0], 1);
    nat::mbar_init(&bars[1], 1);
    nat::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int st = 0; st < 2 && t0 + st < t1; ++st) {
      nat::mbar_arrive_expect_tx(&bars[st], kBytes);
      nat::bulk_g2s(buf + st * kTileD, src + (size_t)(t0 + st) * kTileD, kBytes, &bars[st]);
    }
  }
  for (int it = 0; t0 + it < t1; ++it) {
    const int st = it & 1;
    nat::mbar_wait(&bars[st], (it >> 1) & 1);
    const double2* b2 = reinterpret_cast<const double2*>(buf + st * kTileD);
    for (int s = 0; s < kTile64; ++s) {
      double f[NF];
#pragma unroll
      for (int q = 0; q < NF / 2; ++q) {
        double2 v = b2[s * (NF / 2) + q];
        f[2 * q] = v.x;
        f[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double dx = f[0] - tx[r], dy = f[1] - ty[r], dz = f[2] - tz[r];
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const double dn = fma(dz, f[5], fma(dy, f[4], dx * f[3]));
        // 1/r by rsqrt (MUFU.RSQ64H + Newton) instead of sqrt and a DP division; r = r^2 / r
        const double rho = r2 > 0.0 ? rsqrt(r2) : 0.0;  // self pair (MC operators) -> 0
        const double rr = r2 * rho;
        const double qq = dn * (rho * rho);
        double sn, cs;
        nat::pair_sincos(k * rr, &sn, &cs);
        const double cr = fma(qq, fma(rho, f[6], f[7]), rho * f[10]);
        const double ci = fma(qq, fma(rho, f[9], f[8]), rho * f[11]);
        ar[r] = fma(cs, cr, fma(-sn, ci, ar[r]));
        ai[r] = fma(sn, cr, fma(cs, ci, ai[r]));
      }
    }
    __syncthreads();
    if (tid == 0 && t0 + it + 2 < t1) {
      nat::fence_proxy_async_smem();
      nat::mbar_arrive_expect_tx(&bars[st], kBytes);
      nat::bulk_g2s(buf + st * kTileD, src + (size_t)(t0 + it + 2) * kTileD, kBytes, &bars[st]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t l = tbase + r * kThreads + tid;
    if (l < prm.n_lis && mch < prm.n_modes)
      prm.out[((size_t)split * prm.n_modes + mch) * prm.n_lis + l] = make_double2(ar[r], ai[r]);
  }
}

__global__ void reduce_splits_kernel(const double2* __restrict__ part, int n_split, int64_t n,
                                     double2* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 s = part[i];
  for (int k = 1; k < n_split; ++k) {
    double2 v = part[(size_t)k * n + i];
    s.x += v.x;
    s.y += v.y;
  }
  out[i] = s;
}

struct RuleQ {
  double lam[9], w[3];
  int Q;
};

__global__ void bem_sources_kernel(int64_t nv, int64_t nt, const double* __restrict__ vx,
                                   const int32_t* __restrict__ tri, const double* __restrict__ nrm,
                                   const double* __restrict__ area, RuleQ rq, int n_modes, const double2* __restrict__ p_tri,
                                   const double2* __restrict__ g_tri, double* __restrict__ xyz,
                                   double* __restrict__ nout, double* __restrict__ w,
                                   double2* __restrict__ p_src, double2* __restrict__ g_src) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int Q = rq.Q;
  int64_t S = nt * Q;
  if (i >= S) return;
  int64_t t = i / Q;
  int q = (int)(i % Q);
  int a = tri[t], b = tri[nt + t], c = tri[2 * nt + t];
  double l1 = rq.lam[3 * q], l2 = rq.lam[3 * q + 1], l3 = rq.lam[3 * q + 2];
  for (int d = 0; d < 3; ++d) {
    const double* X = vx + d * nv;
    xyz[d * S + i] = __dadd_rn(__dadd_rn(__dmul_rn(l1, X[a]), __dmul_rn(l2, X[b])), __dmul_rn(l3, X[c]));
    nout[d * S + i] = nrm[d * nt + t];
  }
  w[i] = rq.w[q] * area[t];
  for (int m = 0; m < n_modes; ++m) {
    p_src[(size_t)m * S + i] = p_tri[(size_t)m * nt + t];
    g_src[(size_t)m * S + i] = g_tri[(size_t)m * nt + t];
  }
}

__global__ void mc_sources_kernel(int64_t M, const double* __restrict__ smp, double wv,
                                  double* __restrict__ xyz, double* __restrict__ nrm,
                                  double* __restrict__ w) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  for (int d = 0; d < 3; ++d) {
    xyz[d * M + i] = smp[d * M + i];
    nrm[d * M + i] = smp[(3 + d) * M + i];
  }
  w[i] = wv;
}

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
struct Plan {
  int kind;  // record / kernel kind (fp32 only; see rec_geo)
  int MB, R, NF, n_mchunk, tile, n_tiles, chunk_tiles, n_split, sub = 1;
  int64_t n_src_pad, tgt_tiles;
  size_t rec_elems, smem;
  bool fp64;
  int NT;  // threads per CTA of the fp32 kernel
};

// wavenumbers per launch chunk: up to 8 share r, 1/r and d.n (MUFU 2 + 1/MB per pair-mode);
// NAT_MAX_MB (4 or 8) caps it for A/B comparisons
int pick_mb(int n_modes) {
  static const int cap = [] {
    const char* e = std::getenv("NAT_MAX_MB");
    return (e && std::atoi(e) == 4) ? 4 : 8;
  }();
  if (n_modes >= 8 && cap >= 8) return 8;
  if (n_modes >= 4) return 4;
  if (n_modes == 3) return 3;
  if (n_modes == 2) return 2;
  return 1;
}

template <int R, int MB, int KIND, int NT>
int occ_of(size_t smem) {
  int occ = 0;
  auto k = radiate_f32x2_kernel<R, MB, KIND, NT>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  return occ > 0 ? occ : 1;
}

template <int R, int KIND, int NT>
int occ_mb(int MB, size_t smem) {
  if constexpr (KIND == 1) {  // the MC operator also has balanced chunks of 5-7 wavenumbers
    if (MB == 5) return occ_of<R, 5, KIND, NT>(smem);
    if (MB == 6) return occ_of<R, 6, KIND, NT>(smem);
    if (MB == 7) return occ_of<R, 7, KIND, NT>(smem);
  }
  return MB == 1 ? occ_of<R, 1, KIND, NT>(smem) : MB == 2 ? occ_of<R, 2, KIND, NT>(smem)
       : MB == 3 ? occ_of<R, 3, KIND, NT>(smem) : MB == 4 ? occ_of<R, 4, KIND, NT>(smem)
       : occ_of<R, 8, KIND, NT>(smem);
}
template <int R, int NT>
int occ_kind(int kind, int MB, size_t smem) {
  return kind == 0 ? occ_mb<R, 0, NT>(MB, smem) : kind == 1 ? occ_mb<R, 1, NT>(MB, smem) : occ_mb<R, 2, NT>(MB, smem);
}

// Resident CTAs per SM of the radiation kernel instance (cached per configuration).
int occupancy(bool fp64, int kind, int R, int MB, int NT, size_t smem) {
  static int cache[2][3][5][9][2];  // [fp64][kind][R][MB][NT == 128], 0 = unknown
  int& c = cache[fp64 ? 1 : 0][fp64 ? 0 : kind][R][MB][NT == 128 ? 1 : 0];
  if (c) return c;
  if (fp64) {
    int occ = 0;
    auto k = radiate_f64_kernel<2>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem) != cudaSuccess) {
      cudaGetLastError();
      occ = 2;
    }
    c = occ > 0 ? occ : 1;
  } else if (NT == 128) {
    c = R == 2 ? occ_kind<2, 128>(kind, MB, smem) : occ_kind<4, 128>(kind, MB, smem);
  } else {
    c = R == 2 ? occ_kind<2, 256>(kind, MB, smem) : occ_kind<4, 256>(kind, MB, smem);
  }
  return c;
}

Plan make_plan(nat_prec prec, int64_t n_src, int n_modes, int64_t n_lis, int kind) {
  Plan pl{};
  pl.fp64 = (prec == NAT_FP64);
  pl.kind = pl.fp64 ? 0 : kind;
  if (pl.fp64) {
    pl.MB = 1;
    pl.R = 2;
    pl.NF = 12;
    pl.tile = kTile64;
  } else {
    pl.MB = pick_mb(n_modes);
    // MC operator (the compacted tail launches any n): the same chunk count with balanced
    // chunks, ceil(n / ceil(n / 8)) wavenumbers each, so the last chunk carries no padding
    // (n = 41: 6 x 7 slots instead of 6 x 8); NAT_MB_BALANCE=0 disables (A/B)
    static const bool balance = [] {
      const char* e = std::getenv("NAT_MB_BALANCE");
      return !(e && e[0] == '0');
    }();
    if (balance && kind == 1 && pl.MB == 8) {
      const int chunks = (n_modes + 7) / 8;
      pl.MB = (n_modes + chunks - 1) / chunks;
      if (pl.MB < 5) pl.MB = 8;  // (never: n >= 8 gives 5..8)
    }
    pl.R = 4;
    pl.NF = rec_nf(pl.kind, pl.MB);  // records of the FP32x2 kernel (scalars, broadcast operands)
    pl.tile = kTile;
  }
  pl.NT = kThreads;
  pl.n_mchunk = (n_modes + pl.MB - 1) / pl.MB;
  pl.n_tiles = (int)((n_src + pl.tile - 1) / pl.tile);
  pl.n_src_pad = (int64_t)pl.n_tiles * pl.tile;
  // Choose the CTA width NT, targets/thread R and the source chunk (tiles per CTA,
  // split-K) minimising the modelled time of the busiest SM (all CTAs do equal work).
  const int n_sm = nat::device_sm_count();
  double best = 1e300;
  struct Cand {
    double cost;
    int R, NT;
    int64_t tgt;
    int c;
    size_t smem;
  };
  std::vector<Cand> cands;
  const int r_opts[2] = {4, 2}, nt_opts[2] = {256, 128};
  for (int ni = 0; ni < (pl.fp64 ? 1 : 2); ++ni)
    for (int ri = 0; ri < (pl.fp64 ? 1 : 2); ++ri) {
      const int R = pl.fp64 ? 2 : r_opts[ri];
      const int NT = pl.fp64 ? kThreads : nt_opts[ni];
      const size_t smem = pl.fp64 ? 2 * (size_t)kTile64 * 12 * sizeof(double)
                                  : 2 * (size_t)kTile * pl.NF * sizeof(float);
      const int occ = occupancy(pl.fp64, pl.kind, R, pl.MB, NT, smem);
      const int64_t tgt = (n_lis + (int64_t)R * NT - 1) / ((int64_t)R * NT);
      const int64_t base = tgt * pl.n_mchunk;
      const int tile = pl.fp64 ? kTile64 : kTile;
      // per-SM pair throughput at the MUFU roofline (~1.0e10 pairs/s per SM, fp32)
      const double sm_rate = pl.fp64 ? 1.2e9 : 1.0e10;
      // fp32 kernel: a CTA's source chunk may span more than kMaxChunkTiles tiles (its fp32
      // sums are flushed to fp64 every kMaxChunkTiles tiles)
      const int c_max = pl.n_tiles;
      for (int c = 1; c <= c_max; ++c) {
        const int64_t ns = (pl.n_tiles + c - 1) / c;
        if (c > 1 && (pl.n_tiles + c - 2) / (c - 1) == ns) continue;  // same split count, more work
        // the busiest SM runs cpsm CTAs of work W in rounds of `occ` resident CTAs; a round
        // of r CTAs proceeds at sm_rate * eff(r) (measured, ncu r01: the MUFU/FMA pipes need
        // ~40 resident warps per SM to saturate)
        const int64_t cpsm = (base * ns + n_sm - 1) / n_sm;
        auto eff = [&](int64_t r) { return std::min(1.0, (double)r * (NT / 32) / 40.0); };
        const double W = (double)c * tile * R * NT * pl.MB;
        const int64_t full = cpsm / occ, rest = cpsm % occ;
        double t_comp = (double)full * occ * W / (sm_rate * eff(occ));
        if (rest) t_comp += (double)rest * W / (sm_rate * eff(rest));
        // R = 2 doubles the shared-memory loads per pair; a CTA has a fixed prologue/epilogue
        t_comp *= (R == 2 ? 1.1 : 1.0);
        const double t_fix = (double)(full + (rest > 0)) * 0.5e-6;  // sweep r01: finest splits win on MC shapes
        // split-K partials: written once, read by the epilogue; for the MC operators (small,
        // L2-resident) the kernel-timer sweep (scripts/sweep_mc.py, r01) found the finest
        // split fastest, so their partial traffic is charged at L2 rather than HBM speed
        const double t_part =
            ns > 1 ? (double)ns * n_modes * n_lis * 32.0 / (pl.kind != 0 ? 24.0e12 : 6.0e12) : 0.0;
        const double cost = t_comp + t_fix + t_part + 2e-6 * (ns > 1);
        cands.push_back({cost, R, NT, tgt, c, smem});
        if (cost < best) {
          best = cost;
          pl.R = R;
          pl.NT = NT;
          pl.tgt_tiles = tgt;
          pl.chunk_tiles = c;
          pl.smem = smem;
        }
      }
    }
  // MC operators (targets = sources, ~1e8 pairs per wavenumber): the model cannot see the
  // tail of the last CTA wave; the kernel-timer sweep (scripts/sweep_mc.py, r01: 232 -> 209
  // us at M = 10,000, 3 wavenumbers) favours the finest split among near-equal costs
  static const bool coarse = std::getenv("NAT_MC_COARSE") != nullptr;  // tuning comparisons only
  if (pl.kind != 0 && !pl.fp64 && !coarse) {
    int best_c = pl.chunk_tiles;
    for (const Cand& q : cands)
      if (q.cost <= 1.15 * best && (q.c < best_c || (q.c == best_c && q.R * q.NT < pl.R * pl.NT))) {
        best_c = q.c;
        pl.R = q.R;
        pl.NT = q.NT;
        pl.tgt_tiles = q.tgt;
        pl.chunk_tiles = q.c;
        pl.smem = q.smem;
      }
  }
  if (const char* ov = std::getenv("NAT_RAD_PLAN")) {  // tuning sweeps only: "R,NT,c[,MB[,kind]]"
    int R = 0, NT = 0, c = 0, MB = 0, kd = -1;
    const int nf = pl.fp64 ? 0 : std::sscanf(ov, "%d,%d,%d,%d,%d", &R, &NT, &c, &MB, &kd);
    if (nf >= 3 && (R == 2 || R == 4) && (NT == 128 || NT == 256) && c >= 1 && (kd < 0 || kd == pl.kind)) {
      if (nf >= 4 && (MB == 1 || MB == 2 || MB == 3 || MB == 4 || MB == 8)) {
        pl.MB = MB;
        pl.NF = rec_nf(pl.kind, pl.MB);
        pl.n_mchunk = (n_modes + pl.MB - 1) / pl.MB;
      }
      pl.R = R;
      pl.NT = NT;
      pl.chunk_tiles = std::min(c, pl.n_tiles);
      pl.tgt_tiles = (n_lis + (int64_t)R * NT - 1) / ((int64_t)R * NT);
      pl.smem = 2 * (size_t)kTile * pl.NF * sizeof(float);
    }
  }
  pl.n_split = (pl.n_tiles + pl.chunk_tiles - 1) / pl.chunk_tiles;
  // MC operators whose grid leaves SMs idle (the compacted tail of a solve: few wavenumbers,
  // one tile per CTA already): 2 or 4 CTAs per source tile (NAT_RAD_SUB=0 disables; A/B)
  static const bool sub_on = [] {
    const char* e = std::getenv("NAT_RAD_SUB");
    return !(e && e[0] == '0');
  }();
  if (sub_on && !pl.fp64 && pl.kind != 0 && pl.chunk_tiles == 1) {
    const int64_t ctas = pl.tgt_tiles * pl.n_mchunk * pl.n_split;
    pl.sub = ctas >= 2 * (int64_t)n_sm ? 1 : ctas * 2 >= 2 * (int64_t)n_sm ? 2 : 4;
    pl.n_split *= pl.sub;
  }
  static const bool dbg = std::getenv("NAT_DEBUG_PLAN") != nullptr;
  if (dbg)
    std::fprintf(stderr, "[plan] kind %d modes %d src %lld lis %lld: R %d NT %d MB %d chunk %d split %d (sub %d) tgt %lld occ %d smem %zu\n",
                 pl.kind, n_modes, (long long)n_src, (long long)n_lis, pl.R, pl.NT, pl.MB, pl.chunk_tiles, pl.n_split, pl.sub,
                 (long long)pl.tgt_tiles, occupancy(pl.fp64, pl.kind, pl.R, pl.MB, pl.NT, pl.smem), pl.smem);
  pl.rec_elems = (size_t)pl.n_mchunk * pl.n_src_pad * pl.NF;
  return pl;
}

size_t plan_ws(const Plan& pl, int n_modes, int64_t n_lis, nat::Carver& c, void** rec, double2** part) {
  *rec = pl.fp64 ? (void*)c.take<double>(pl.rec_elems) : (void*)c.take<float>(pl.rec_elems);
  *part = pl.n_split > 1 ? c.take<double2>((size_t)pl.n_split * n_modes * n_lis) : nullptr;
  return c.bytes();
}

template <int R, int MB, int KIND, int NT>
cudaError_t launch_f32(const Plan& pl, const RadParams& prm, cudaStream_t s) {
  auto kern = radiate_f32x2_kernel<R, MB, KIND, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)pl.tgt_tiles, (unsigned)pl.n_split, (unsigned)pl.n_mchunk);
  kern<<<grid, NT, pl.smem, s>>>(prm);
  return cudaGetLastError();
}

template <int R, int KIND, int NT>
cudaError_t launch_f32_r(const Plan& pl, const RadParams& prm, cudaStream_t s) {
  switch (pl.MB) {
    case 1: return launch_f32<R, 1, KIND, NT>(pl, prm, s);
    case 2: return launch_f32<R, 2, KIND, NT>(pl, prm, s);
    case 3: return launch_f32<R, 3, KIND, NT>(pl, prm, s);
    case 4: return launch_f32<R, 4, KIND, NT>(pl, prm, s);
    case 5: if constexpr (KIND == 1) return launch_f32<R, 5, KIND, NT>(pl, prm, s); else break;
    case 6: if constexpr (KIND == 1) return launch_f32<R, 6, KIND, NT>(pl, prm, s); else break;
    case 7: if constexpr (KIND == 1) return launch_f32<R, 7, KIND, NT>(pl, prm, s); else break;
    default: break;
  }
  return launch_f32<R, 8, KIND, NT>(pl, prm, s);
}

template <int KIND>
cudaError_t launch_f32_mb(const Plan& pl, const RadParams& prm, cudaStream_t s) {
  if (pl.NT == 128)
    return pl.R == 2 ? launch_f32_r<2, KIND, 128>(pl, prm, s) : launch_f32_r<4, KIND, 128>(pl, prm, s);
  return pl.R == 2 ? launch_f32_r<2, KIND, 256>(pl, prm, s) : launch_f32_r<4, KIND, 256>(pl, prm, s);
}

}  // namespace

namespace nat {

// The launch shape for n_lis targets, chosen as for plan_lis targets when plan_lis > 0.
Plan plan_for(nat_prec prec, int64_t n_src, int nm, int64_t n_lis, int kind, int64_t plan_lis) {
  Plan pl = make_plan(prec, n_src, nm, plan_lis > 0 ? plan_lis : n_lis, kind);
  pl.tgt_tiles = (n_lis + (int64_t)pl.R * pl.NT - 1) / ((int64_t)pl.R * pl.NT);
  return pl;
}

size_t radiate_ws_bytes(nat_prec prec, int64_t n_src, int n_modes, int64_t n_lis, int kind, int64_t plan_lis) {
  if (n_src <= 0 || n_modes <= 0 || n_lis <= 0) return 0;
  const int nm = n_modes < kMaxModes ? n_modes : kMaxModes;
  Plan pl = plan_for(prec, n_src, nm, n_lis, kind, plan_lis);
  Carver c(nullptr);
  void* rec;
  double2* part;
  return plan_ws(pl, nm, n_lis, c, &rec, &part);
}

size_t radiate_ws_bytes_upto(nat_prec prec, int64_t n_src, int max_modes, int64_t n_lis) {
  size_t b = 0;
  for (int m = 1; m <= (max_modes < kMaxModes ? max_modes : kMaxModes); ++m)
    for (int kind = 0; kind < 3; ++kind) b = std::max(b, radiate_ws_bytes(prec, n_src, m, n_lis, kind));
  return b;
}

nat_status radiate_internal(const RadInput& in, nat_prec prec, const double* k, int64_t n_lis,
                            const double* lis, double2* out, void* ws, size_t ws_bytes, bool self,
                            cudaStream_t s, RadPartials* keep) {
  if (keep && in.n_modes > kMaxModes) return fail(NAT_ERR_INVALID_ARG, "unreduced partials need <= 64 modes");
  // self-excluding launches are the MC operators: double layer (g absent) or single layer (p absent)
  if (self && in.p && in.g) return fail(NAT_ERR_INVALID_ARG, "self-excluding radiation needs p or g absent");
  const int kind = !self ? 0 : (in.p ? 1 : 2);
  for (int m0 = 0; m0 < in.n_modes; m0 += kMaxModes) {
    const int nm = (in.n_modes - m0) < kMaxModes ? (in.n_modes - m0) : kMaxModes;
    Plan pl = plan_for(prec, in.n_src, nm, n_lis, kind, in.plan_lis);
    Carver c(ws);
    void* rec;
    double2* part;
    size_t need = plan_ws(pl, nm, n_lis, c, &rec, &part);
    if (ws_bytes < need) return fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
    KVals kv{};
    for (int m = 0; m < nm; ++m) {
      kv.d[m] = k[m0 + m];
      kv.f[m] = (float)kv.d[m];
    }
    const double2* p = in.p ? in.p + (size_t)m0 * in.ldpg : nullptr;
    const double2* g = in.g ? in.g + (size_t)m0 * in.ldpg : nullptr;
    const dim3 sblocks((unsigned)((pl.n_src_pad + kStageSrc - 1) / kStageSrc), (unsigned)pl.n_mchunk);
    if (pl.fp64)
      stage_kernel<double><<<sblocks, kStageSrc, 0, s>>>(in.n_src, pl.n_src_pad, pl.NF, pl.MB, pl.n_mchunk, 0,
          in.xyz, in.nrm, in.w, in.w_const, p, g, in.ldpg, kv, nm, in.center[0], in.center[1],
          in.center[2], (double*)rec, in.skip);
    else
      stage_kernel<float, false, -1><<<sblocks, kStageSrc, 0, s>>>(in.n_src, pl.n_src_pad, pl.NF, pl.MB, pl.n_mchunk, pl.kind,
          in.xyz, in.nrm, in.w, in.w_const, p, g, in.ldpg, kv, nm, in.center[0], in.center[1],
          in.center[2], (float*)rec, in.skip);
    NAT_LAUNCH_CHECK();
    RadParams prm{};
    prm.rec = rec;
    prm.n_src_pad = pl.n_src_pad;
    prm.n_tiles = pl.n_tiles;
    prm.chunk_tiles = pl.chunk_tiles;
    prm.lis = lis;
    prm.n_lis = n_lis;
    prm.cx = in.center[0];
    prm.cy = in.center[1];
    prm.cz = in.center[2];
    prm.k = kv;
    double2* dst = out + (size_t)m0 * n_lis;
    prm.out = pl.n_split > 1 ? part : dst;
    prm.n_modes = nm;
    prm.self_r2 = in.self_r2;
    prm.skip = in.skip;
    prm.sub = pl.fp64 ? 1 : pl.sub;
    cudaError_t e = cudaSuccess;
    const int tcat = kind == 0 ? kTimerRadiate : kind == 1 ? kTimerMcOp : kTimerMcRhs;
    const bool timed = ktimer_on();
    if (timed) ktimer_begin(tcat, s);
    if (pl.fp64) {
      auto kern = radiate_f64_kernel<2>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
      if (e == cudaSuccess) {
        dim3 grid((unsigned)pl.tgt_tiles, (unsigned)pl.n_split, (unsigned)pl.n_mchunk);
        kern<<<grid, kThreads, pl.smem, s>>>(prm);
        e = cudaGetLastError();
      }
    } else {
      e = kind == 0 ? launch_f32_mb<0>(pl, prm, s) : kind == 1 ? launch_f32_mb<1>(pl, prm, s)
                                                   : launch_f32_mb<2>(pl, prm, s);
    }
    if (e != cudaSuccess) return fail(NAT_ERR_CUDA, "radiate launch: %s", cudaGetErrorString(e));
    if (timed)  // algorithmic pairs: the self kinds skip the diagonal
      ktimer_end(tcat, s, (double)nm * (double)n_lis * (double)(self ? in.n_src - 1 : in.n_src), in.skip, nm);
    if (keep) {  // the caller reduces the partials in its own epilogue
      keep->part = pl.n_split > 1 ? part : dst;
      keep->n_split = pl.n_split;
    } else if (pl.n_split > 1) {
      int64_t n = (int64_t)nm * n_lis;
      reduce_splits_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(part, pl.n_split, n, dst);
      NAT_LAUNCH_CHECK();
    }
  }
  return NAT_OK;
}

}  // namespace nat

extern "C" size_t nat_radiate_workspace(nat_prec prec, int64_t n_src, int n_modes, int64_t n_lis) {
  return nat::radiate_ws_bytes(prec, n_src, n_modes, n_lis);
}

extern "C" nat_status nat_radiate_field(const nat_sources* src, nat_prec prec, const double* k,
                                        int64_t n_lis, const double* lis_xyz, void* p_out, void* ws,
                                        size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(src && k, "src and k must be non-null");
  NAT_REQUIRE(prec == NAT_FP32 || prec == NAT_FP64, "bad precision %d", (int)prec);
  NAT_REQUIRE(src->n_src > 0 && src->n_modes > 0 && n_lis > 0, "need n_src, n_modes, n_lis > 0");
  NAT_REQUIRE(src->n_src < (1LL << 31) && n_lis < (1LL << 40), "size out of range");
  for (int m = 0; m < src->n_modes; ++m)
    NAT_REQUIRE(k[m] >= 0.0 && k[m] < 1e300, "k[%d] = %g must be finite and >= 0", m, k[m]);
  NAT_REQUIRE_DEV(src->xyz);
  NAT_REQUIRE_DEV(src->nrm);
  NAT_REQUIRE_DEV(src->w);
  NAT_REQUIRE_DEV(src->p);
  NAT_REQUIRE_DEV(src->g);
  NAT_REQUIRE_DEV(lis_xyz);
  NAT_REQUIRE_DEV(p_out);
  NAT_REQUIRE_DEV(ws);
  nat::RadInput in{};
  in.n_src = src->n_src;
  in.xyz = src->xyz;
  in.nrm = src->nrm;
  in.w = src->w;
  in.n_modes = src->n_modes;
  in.p = (const double2*)src->p;
  in.g = (const double2*)src->g;
  in.ldpg = src->n_src;
  for (int d = 0; d < 3; ++d) in.center[d] = src->center[d];
  return nat::radiate_internal(in, prec, k, n_lis, lis_xyz, (double2*)p_out, ws, ws_bytes, false,
                               (cudaStream_t)stream);
}

namespace {
// Barycentric rules for the radiation sources (the library's own tables).
bool rad_rule(int q, double* lam, double* w) {
  switch (q) {
    case 1:
      lam[0] = lam[1] = lam[2] = 1.0 / 3.0;
      w[0] = 1.0;
      return true;
    case 3: {
      const double a = 2.0 / 3.0, b = 1.0 / 6.0;
      double L[9] = {a, b, b, b, a, b, b, b, a};
      for (int i = 0; i < 9; ++i) lam[i] = L[i];
      w[0] = w[1] = w[2] = 1.0 / 3.0;
      return true;
    }
    default:
      return false;
  }
}
}  // namespace

extern "C" nat_status nat_bem_sources(const nat_mesh* mesh, const nat_geom* geom, int q_rad,
                                      int n_modes, const void* p_tri, const void* g_tri, double* xyz,
                                      double* nrm, double* w, void* p_src, void* g_src,
                                      nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(mesh && geom, "mesh and geom must be non-null");
  if (q_rad == 0) q_rad = 3;
  double lam[9], wq[3];
  NAT_REQUIRE(rad_rule(q_rad, lam, wq), "q_rad must be 1 or 3 (got %d)", q_rad);
  NAT_REQUIRE(n_modes >= 1, "n_modes must be >= 1");
  NAT_REQUIRE_DEV(mesh->vxyz);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->normal);
  NAT_REQUIRE_DEV(geom->area);
  NAT_REQUIRE_DEV(p_tri);
  NAT_REQUIRE_DEV(g_tri);
  NAT_REQUIRE_DEV(xyz);
  NAT_REQUIRE_DEV(nrm);
  NAT_REQUIRE_DEV(w);
  NAT_REQUIRE_DEV(p_src);
  NAT_REQUIRE_DEV(g_src);
  cudaStream_t s = (cudaStream_t)stream;
  RuleQ rq{};
  rq.Q = q_rad;
  for (int i = 0; i < 3 * q_rad; ++i) rq.lam[i] = lam[i];
  for (int i = 0; i < q_rad; ++i) rq.w[i] = wq[i];
  int64_t S = mesh->n_tri * q_rad;
  bem_sources_kernel<<<(unsigned)((S + 255) / 256), 256, 0, s>>>(
      mesh->n_vert, mesh->n_tri, mesh->vxyz, mesh->tri, geom->normal, geom->area, rq, n_modes, (const double2*)p_tri, (const double2*)g_tri, xyz, nrm, w,
      (double2*)p_src, (double2*)g_src);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

extern "C" nat_status nat_mc_sources(int64_t M, const double* samples, double total_area, double* xyz,
                                     double* nrm, double* w, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(M >= 1 && total_area > 0, "need M >= 1 and total_area > 0");
  NAT_REQUIRE_DEV(samples);
  NAT_REQUIRE_DEV(xyz);
  NAT_REQUIRE_DEV(nrm);
  NAT_REQUIRE_DEV(w);
  mc_sources_kernel<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      M, samples, total_area / (double)M, xyz, nrm, w);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
