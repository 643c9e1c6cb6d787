// NEXT-3 — Poisson-disk boundary samples on the GPU ("parallel Poisson disk
// sampling [bowers2010]"; l.402 ~10 ms against ~1 ms for random sampling; reading
// R-poisson).
//
// Phase-group dart throwing over a fixed candidate pool, identical (bitwise, index for
// index) to oracle/poisson.py:
//   candidates  30 M_target points of the a8 construction with Philox tag 2;
//   grid        cells of size h = r / sqrt(3) over centre +- R (dense; a cell holds at
//               most one sample, conflicts only inside the 5^3 neighbourhood, cells of one
//               phase (i mod 3 per axis) never conflict);
//   trials      for t = 0, 1, ..., max cell count - 1 and phase p = 0..26, every empty
//               cell of phase p with more than t candidates tests its t-th candidate
//               (ascending index) against the accepted samples of its neighbourhood
//               (fp64, each op rounded, no FMA) — one launch per (t, p), cells of the
//               phase in parallel (the result does not depend on their order);
//   output      the accepted candidates ascending by candidate index.
// The per-cell candidate lists come from a counting sort (atomic fill, then each cell's
// short list sorted by index), so every intermediate is deterministic.
#include <cmath>
#include <vector>

#include "nat_internal.cuh"
#include "sampling.cuh"

namespace {

constexpr int kNCandPerTarget = 30;
constexpr int kT = 256;

struct Grid {
  double ox, oy, oz, h;
  int64_t n;  // cells per axis
};

__device__ __forceinline__ int64_t axis_cell(double x, double o, double h, int64_t n) {
  const double q = floor(__ddiv_rn(__dsub_rn(x, o), h));
  int64_t i = (int64_t)q;
  if (q < 0.0) i = 0;
  if (i > n - 1) i = n - 1;
  return i;
}

__global__ void cell_count_kernel(int64_t nc, const double* __restrict__ cand, Grid g, int32_t* __restrict__ ckey,
                                  int32_t* __restrict__ cnt) {
  const int64_t c = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (c >= nc) return;
  const int64_t ix = axis_cell(cand[c], g.ox, g.h, g.n), iy = axis_cell(cand[nc + c], g.oy, g.h, g.n),
                iz = axis_cell(cand[2 * nc + c], g.oz, g.h, g.n);
  const int32_t key = (int32_t)((iz * g.n + iy) * g.n + ix);
  ckey[c] = key;
  atomicAdd(&cnt[key], 1);
}

__global__ void cell_fill_kernel(int64_t nc, const int32_t* __restrict__ ckey, const int32_t* __restrict__ start,
                                 int32_t* __restrict__ fill, int32_t* __restrict__ lists) {
  const int64_t c = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (c >= nc) return;
  const int32_t key = ckey[c];
  lists[start[key] + atomicAdd(&fill[key], 1)] = (int32_t)c;
}

// Sorts each non-empty cell's list by candidate index, tracks the largest count and
// buckets the non-empty cells by phase (order inside a bucket is irrelevant).
__global__ void cell_finish_kernel(int64_t G, int64_t n, const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ start, int32_t* __restrict__ lists,
                                   int32_t* __restrict__ maxcnt, int32_t* __restrict__ phase_cnt) {
  const int64_t key = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (key >= G) return;
  const int32_t k = cnt[key];
  if (k == 0) return;
  int32_t* l = lists + start[key];
  for (int a = 1; a < k; ++a) {  // insertion sort (a handful of entries)
    const int32_t v = l[a];
    int b = a - 1;
    while (b >= 0 && l[b] > v) {
      l[b + 1] = l[b];
      --b;
    }
    l[b + 1] = v;
  }
  atomicMax(maxcnt, k);
  const int64_t ix = key % n, iy = (key / n) % n, iz = key / (n * n);
  atomicAdd(&phase_cnt[(ix % 3) + 3 * (iy % 3) + 9 * (iz % 3)], 1);
}

__global__ void phase_offsets_kernel(const int32_t* __restrict__ phase_cnt, int32_t* __restrict__ phase_off) {
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int p = 0; p < 27; ++p) {
      phase_off[p] = acc;
      acc += phase_cnt[p];
    }
    phase_off[27] = acc;
  }
}

__global__ void phase_fill_kernel(int64_t G, int64_t n, const int32_t* __restrict__ cnt,
                                  const int32_t* __restrict__ phase_off, int32_t* __restrict__ phase_cur,
                                  int32_t* __restrict__ phase_cells) {
  const int64_t key = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (key >= G || cnt[key] == 0) return;
  const int64_t ix = key % n, iy = (key / n) % n, iz = key / (n * n);
  const int p = (int)((ix % 3) + 3 * (iy % 3) + 9 * (iz % 3));
  phase_cells[phase_off[p] + atomicAdd(&phase_cur[p], 1)] = (int32_t)key;
}

// Trial t of one phase: each listed cell (all of the same phase) tests its t-th candidate.
__global__ void trial_kernel(int ncell, const int32_t* __restrict__ cells, int t, int64_t n, int64_t nc,
                             const double* __restrict__ cand, const int32_t* __restrict__ cnt,
                             const int32_t* __restrict__ start, const int32_t* __restrict__ lists, double r2,
                             int32_t* __restrict__ acc) {
  const int i = blockIdx.x * kT + threadIdx.x;
  if (i >= ncell) return;
  const int64_t key = cells[i];
  if (acc[key] >= 0 || cnt[key] <= t) return;
  const int32_t c = lists[start[key] + t];
  const double x = cand[c], y = cand[nc + c], z = cand[2 * nc + c];
  const int64_t ix = key % n, iy = (key / n) % n, iz = key / (n * n);
  for (int64_t dz = -2; dz <= 2; ++dz) {
    const int64_t cz = iz + dz;
    if (cz < 0 || cz >= n) continue;
    for (int64_t dy = -2; dy <= 2; ++dy) {
      const int64_t cy = iy + dy;
      if (cy < 0 || cy >= n) continue;
      for (int64_t dx = -2; dx <= 2; ++dx) {
        const int64_t cx = ix + dx;
        if (cx < 0 || cx >= n) continue;
        const int32_t a = acc[(cz * n + cy) * n + cx];
        if (a < 0) continue;
        const double ex = __dsub_rn(x, cand[a]), ey = __dsub_rn(y, cand[nc + a]), ez = __dsub_rn(z, cand[2 * nc + a]);
        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
        if (d2 < r2) return;  // conflict
      }
    }
  }
  acc[key] = c;
}

__global__ void flag_kernel(int64_t G, const int32_t* __restrict__ acc, int32_t* __restrict__ flag) {
  const int64_t key = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (key >= G) return;
  const int32_t a = acc[key];
  if (a >= 0) flag[a] = 1;
}

__global__ void out_kernel(int64_t nc, int64_t M, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                           const double* __restrict__ cand, const int32_t* __restrict__ ctri,
                           double* __restrict__ smp, int32_t* __restrict__ stri) {
  const int64_t c = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (c >= nc || !flag[c]) return;
  const int64_t j = pos[c];
#pragma unroll
  for (int d = 0; d < 6; ++d) smp[d * M + j] = cand[d * nc + c];
  stri[j] = ctri[c];
}

// ---- device-wide exclusive scan of int32 (fixed segmentation, exact) -------------------
constexpr int kScanItems = 4;
constexpr int kScanBlock = 1024 * kScanItems;

__global__ void __launch_bounds__(1024) scan_blocks_kernel(const int32_t* __restrict__ in, int64_t n,
                                                           int32_t* __restrict__ out, int64_t* __restrict__ bsum) {
  __shared__ int64_t sh[33];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + threadIdx.x * kScanItems;
  int64_t v[kScanItems], s = 0;
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    v[u] = base + u < n ? in[base + u] : 0;
    s += v[u];
  }
  int64_t total = 0;
  int64_t acc = nat::block_exscan_1024(s, sh, &total);
#pragma unroll
  for (int u = 0; u < kScanItems; ++u) {
    if (base + u < n) out[base + u] = (int32_t)acc;
    acc += v[u];
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(int64_t* __restrict__ bsum, int64_t nb,
                                                         int64_t* __restrict__ total) {
  __shared__ int64_t sh[33];
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < nb ? bsum[b] : 0;
    int64_t t = 0;
    const int64_t e = nat::block_exscan_1024(v, sh, &t);
    if (b < nb) bsum[b] = carry + e;
    carry += t;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_add_kernel(int32_t* __restrict__ out, int64_t n, const int64_t* __restrict__ bsum) {
  const int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (i >= n) return;
  out[i] += (int32_t)bsum[i / kScanBlock];
}

void scan_i32(const int32_t* in, int64_t n, int32_t* out, int64_t* bsum, int64_t* total, cudaStream_t s) {
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  scan_blocks_kernel<<<(unsigned)nb, 1024, 0, s>>>(in, n, out, bsum);
  scan_sums_kernel<<<1, 1024, 0, s>>>(bsum, nb, total);
  scan_add_kernel<<<(unsigned)((n + kT - 1) / kT), kT, 0, s>>>(out, n, bsum);
}

struct PoissonPlan {
  double r;
  int64_t n_cand;
  Grid g;
  int64_t G;
};

nat_status plan_of(const nat_geom* geom, int64_t M_target, double r, PoissonPlan* p) {
  NAT_REQUIRE(geom, "geom must be non-null");
  NAT_REQUIRE(M_target >= 1 && M_target <= (1LL << 31) / kNCandPerTarget, "M_target out of range");
  NAT_REQUIRE(geom->total_area > 0 && geom->bound_radius > 0, "geom must come from nat_mesh_prepare");
  p->r = r > 0 ? r : 0.7 * std::sqrt(geom->total_area / (double)M_target);
  p->n_cand = kNCandPerTarget * M_target;
  const double R = geom->bound_radius;
  p->g.h = p->r / std::sqrt(3.0);
  p->g.n = (int64_t)std::floor(2.0 * R / p->g.h) + 1;
  p->g.ox = geom->center[0] - R;
  p->g.oy = geom->center[1] - R;
  p->g.oz = geom->center[2] - R;
  NAT_REQUIRE(p->g.n <= 1280, "radius %g too small for the dense cell grid (%lld cells per axis)", p->r,
              (long long)p->g.n);
  p->G = p->g.n * p->g.n * p->g.n;
  return NAT_OK;
}

struct PoissonWs {
  double* cand;       // [6][n_cand]
  int32_t* ctri;      // [n_cand]
  int32_t* ckey;      // [n_cand]
  int32_t* lists;     // [n_cand]
  int32_t* flag;      // [n_cand]
  int32_t* pos;       // [n_cand]
  int32_t* cnt;       // [G]
  int32_t* start;     // [G]
  int32_t* fill;      // [G]
  int32_t* acc;       // [G]
  int32_t* phase_cells;  // [min(G, n_cand)]
  int32_t* small;     // maxcnt, phase_cnt[27], phase_off[28], phase_cur[27]
  int64_t* bsum;      // scan block sums
  int64_t* total;     // [1]
};

size_t carve(nat::Carver& c, const PoissonPlan& p, PoissonWs* w) {
  const int64_t big = p.G > p.n_cand ? p.G : p.n_cand;
  PoissonWs t;
  t.cand = c.take<double>(6 * (size_t)p.n_cand);
  t.ctri = c.take<int32_t>(p.n_cand);
  t.ckey = c.take<int32_t>(p.n_cand);
  t.lists = c.take<int32_t>(p.n_cand);
  t.flag = c.take<int32_t>(p.n_cand);
  t.pos = c.take<int32_t>(p.n_cand);
  t.cnt = c.take<int32_t>(p.G);
  t.start = c.take<int32_t>(p.G);
  t.fill = c.take<int32_t>(p.G);
  t.acc = c.take<int32_t>(p.G);
  t.phase_cells = c.take<int32_t>(p.G < p.n_cand ? p.G : p.n_cand);
  t.small = c.take<int32_t>(1 + 27 + 28 + 27);
  t.bsum = c.take<int64_t>((big + kScanBlock - 1) / kScanBlock + 1);
  t.total = c.take<int64_t>(1);
  if (w) *w = t;
  return c.bytes();
}

}  // namespace

extern "C" size_t nat_mc_poisson_workspace(const nat_geom* geom, int64_t M_target, double r) {
  PoissonPlan p;
  if (plan_of(geom, M_target, r, &p) != NAT_OK) return 0;
  nat::Carver c(nullptr);
  return carve(c, p, nullptr);
}

extern "C" nat_status nat_mc_poisson_sample(const nat_mesh* mesh, const nat_geom* geom, int64_t M_target, double r,
                                            uint64_t seed, uint64_t stream_id, double* samples_out,
                                            int32_t* sample_tri_out, int64_t cap, int64_t* M_out, double* r_out,
                                            void* ws, size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(mesh && geom && M_out, "mesh, geom and M_out must be non-null");
  NAT_REQUIRE(geom->n_tri == mesh->n_tri && mesh->n_tri >= 1, "inconsistent n_tri");
  PoissonPlan p;
  nat_status st = plan_of(geom, M_target, r, &p);
  if (st != NAT_OK) return st;
  NAT_REQUIRE(cap >= 1, "cap must be >= 1");
  NAT_REQUIRE_DEV(mesh->vxyz);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->normal);
  NAT_REQUIRE_DEV(geom->area_cdf);
  NAT_REQUIRE_DEV(samples_out);
  NAT_REQUIRE_DEV(sample_tri_out);
  NAT_REQUIRE_DEV(ws);
  nat::Carver c(ws);
  PoissonWs w;
  const size_t need = carve(c, p, &w);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nc = p.n_cand, G = p.G;
  int32_t* maxcnt = w.small;
  int32_t* phase_cnt = w.small + 1;
  int32_t* phase_off = w.small + 28;
  int32_t* phase_cur = w.small + 56;
  // 1. candidate pool (a8 construction, Philox tag 2)
  st = nat::mc_sample_tagged(mesh, geom, nc, seed, stream_id, 2u, w.cand, w.ctri, s);
  if (st != NAT_OK) return st;
  // 2. counting sort of the candidates into cells
  NAT_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * G, s));
  NAT_CUDA_TRY(cudaMemsetAsync(w.fill, 0, sizeof(int32_t) * G, s));
  NAT_CUDA_TRY(cudaMemsetAsync(w.acc, 0xff, sizeof(int32_t) * G, s));
  NAT_CUDA_TRY(cudaMemsetAsync(w.small, 0, sizeof(int32_t) * (1 + 27 + 28 + 27), s));
  const unsigned gc = (unsigned)((nc + kT - 1) / kT), gg = (unsigned)((G + kT - 1) / kT);
  cell_count_kernel<<<gc, kT, 0, s>>>(nc, w.cand, p.g, w.ckey, w.cnt);
  scan_i32(w.cnt, G, w.start, w.bsum, w.total, s);
  cell_fill_kernel<<<gc, kT, 0, s>>>(nc, w.ckey, w.start, w.fill, w.lists);
  cell_finish_kernel<<<gg, kT, 0, s>>>(G, p.g.n, w.cnt, w.start, w.lists, maxcnt, phase_cnt);
  phase_offsets_kernel<<<1, 32, 0, s>>>(phase_cnt, phase_off);
  phase_fill_kernel<<<gg, kT, 0, s>>>(G, p.g.n, w.cnt, phase_off, phase_cur, w.phase_cells);
  NAT_LAUNCH_CHECK();
  int32_t hs[1 + 27 + 28];
  NAT_CUDA_TRY(cudaMemcpyAsync(hs, w.small, sizeof hs, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  const int T = hs[0];
  const int32_t* off = hs + 28;
  // 3. trials x phases
  const double r2 = p.r * p.r;
  for (int t = 0; t < T; ++t)
    for (int ph = 0; ph < 27; ++ph) {
      const int ncell = off[ph + 1] - off[ph];
      if (ncell > 0)
        trial_kernel<<<(unsigned)((ncell + kT - 1) / kT), kT, 0, s>>>(ncell, w.phase_cells + off[ph], t, p.g.n, nc,
                                                                       w.cand, w.cnt, w.start, w.lists, r2, w.acc);
    }
  NAT_LAUNCH_CHECK();
  // 4. accepted candidates, ascending by index
  NAT_CUDA_TRY(cudaMemsetAsync(w.flag, 0, sizeof(int32_t) * nc, s));
  flag_kernel<<<gg, kT, 0, s>>>(G, w.acc, w.flag);
  scan_i32(w.flag, nc, w.pos, w.bsum, w.total, s);
  NAT_LAUNCH_CHECK();
  int64_t M = 0;
  NAT_CUDA_TRY(cudaMemcpyAsync(&M, w.total, sizeof M, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  *M_out = M;
  if (r_out) *r_out = p.r;
  if (M > cap) return nat::fail(NAT_ERR_WORKSPACE, "%lld Poisson samples > cap %lld", (long long)M, (long long)cap);
  out_kernel<<<gc, kT, 0, s>>>(nc, M, w.flag, w.pos, w.cand, w.ctri, samples_out, sample_tri_out);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
