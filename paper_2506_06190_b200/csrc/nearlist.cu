// Row a2 — near list for the dense BEM ("integrations involving adjacent or
// identical elements"; reading R-near).
//
// For row i (global index) and source triangle j != i:
//   class 1 (S): T_j shares a vertex index with T_i,
//   class 2 (N): otherwise, if sqrt((dx*dx + dy*dy) + dz*dz) < eta*diam_j, d = c_i - c_j,
// evaluated in fp64 with explicit round-to-nearest intrinsics (no FMA contraction), so
// the integer result is identical to the oracle's.  CSR, columns ascending.
//
// Kernels: a prep pass writes, per source tile of 256 triangles, the fp32 bounding box
// of the centroids and the largest reach max(eta diam_j, diam_j) (workspace).  CTA = 8
// warps x 4 rows; the CTA tests every tile's box against its rows' box in parallel,
// compacts the surviving tiles in ascending order, stages only those in shared memory,
// and each warp scans its rows' candidates 32 at a time, compacting hits with
// __ballot_sync (ascending order is preserved).
#include "nat_internal.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kRowsPerWarp = 4;
constexpr int kRowsPerCta = kWarps * kRowsPerWarp;
constexpr int kJTile = 256;

struct TileBox {  // fp32, conservative
  float lo[3], hi[3], reach, pad;
};

struct NearArgs {
  int64_t nt, row_begin, rows;
  const int32_t* tri;
  const double* cen;
  const double* diam;
  double eta;
  const TileBox* tbox;     // [n_tiles]
  int n_tiles;
  const int64_t* row_ptr;  // build pass: offsets (relative to row_begin)
  int64_t* counts;         // count pass: counts[r + 1]
  int32_t* col;
  uint8_t* cls;
};

__global__ void __launch_bounds__(kJTile) tile_box_kernel(int64_t nt, const double* __restrict__ cen,
                                                         const double* __restrict__ diam, double eta,
                                                         TileBox* __restrict__ tb) {
  __shared__ float red[kJTile / 32][7];
  const int64_t j = (int64_t)blockIdx.x * kJTile + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float v[7];
  if (j < nt) {
    const float c[3] = {(float)cen[j], (float)cen[nt + j], (float)cen[2 * nt + j]};
    for (int d = 0; d < 3; ++d) {
      v[d] = c[d];
      v[3 + d] = -c[d];
    }
    v[6] = -fmaxf((float)__dmul_rn(eta, diam[j]), (float)diam[j]);
  } else {
    for (int d = 0; d < 6; ++d) v[d] = 3e30f;
    v[6] = 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 7; ++c) v[c] = fminf(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
  if (lane == 0)
    for (int c = 0; c < 7; ++c) red[warp][c] = v[c];
  __syncthreads();
  if (threadIdx.x == 0) {
    float b[7];
    for (int c = 0; c < 7; ++c) {
      b[c] = red[0][c];
      for (int w = 1; w < kJTile / 32; ++w) b[c] = fminf(b[c], red[w][c]);
    }
    TileBox t;
    for (int d = 0; d < 3; ++d) {
      t.lo[d] = b[d];
      t.hi[d] = -b[3 + d];
    }
    t.reach = -b[6];
    t.pad = 0.f;
    tb[blockIdx.x] = t;
  }
}

template <bool kBuild>
__global__ void __launch_bounds__(kWarps * 32) near_kernel(NearArgs a) {
  __shared__ double s_cx[kJTile], s_cy[kJTile], s_cz[kJTile], s_thr[kJTile];
  __shared__ float s_f[5][kJTile];  // fp32 centroid, eta*diam, diam: conservative prefilter
  __shared__ int32_t s_v[3][kJTile];
  __shared__ int s_live[kJTile];    // surviving tiles of the current chunk, ascending
  __shared__ int s_nlive;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta + warp * kRowsPerWarp;
  const int64_t nt = a.nt;

  // the rows' fp64 centroids live in shared memory (used only by the exact test, rarely)
  __shared__ double s_rc[kWarps][kRowsPerWarp][3];
  __shared__ float s_rd[kWarps][kRowsPerWarp];
  __shared__ float s_rb[8];            // rows: min xyz, -max xyz, max diam, fp32 margin
  int64_t gi[kRowsPerWarp];
  float fx[kRowsPerWarp], fy[kRowsPerWarp], fz[kRowsPerWarp], fd[kRowsPerWarp];
  int32_t va[kRowsPerWarp], vb[kRowsPerWarp], vc[kRowsPerWarp];
  int64_t pos[kRowsPerWarp];
  bool live[kRowsPerWarp];
#pragma unroll
  for (int q = 0; q < kRowsPerWarp; ++q) {
    int64_t r = r0 + q;
    live[q] = r < a.rows;
    int64_t i = a.row_begin + (live[q] ? r : 0);
    gi[q] = i;
    const double cxd = a.cen[i], cyd = a.cen[nt + i], czd = a.cen[2 * nt + i];
    if (lane == 0) {
      s_rc[warp][q][0] = cxd;
      s_rc[warp][q][1] = cyd;
      s_rc[warp][q][2] = czd;
      s_rd[warp][q] = live[q] ? (float)a.diam[i] : -1.f;
    }
    fx[q] = (float)cxd;
    fy[q] = (float)cyd;
    fz[q] = (float)czd;
    fd[q] = (float)a.diam[i];
    va[q] = a.tri[i];
    vb[q] = a.tri[nt + i];
    vc[q] = a.tri[2 * nt + i];
    pos[q] = (kBuild && live[q]) ? a.row_ptr[r] : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // bounding box of this CTA's live rows (fp32, for tile skipping)
    float b[7] = {3e30f, 3e30f, 3e30f, 3e30f, 3e30f, 3e30f, 0.f};
    float mabs = 0.f;
    for (int w = 0; w < kWarps; ++w)
      for (int q = 0; q < kRowsPerWarp; ++q) {
        if (s_rd[w][q] < 0.f) continue;
        for (int d = 0; d < 3; ++d) {
          const float c = (float)s_rc[w][q][d];
          b[d] = fminf(b[d], c);
          b[3 + d] = fminf(b[3 + d], -c);
          mabs = fmaxf(mabs, fabsf(c));
        }
        b[6] = fmaxf(b[6], s_rd[w][q]);
      }
    for (int c = 0; c < 7; ++c) s_rb[c] = b[c];
    s_rb[7] = 1e-5f * (1.f + mabs);
  }
  __syncthreads();

  for (int tc = 0; tc < a.n_tiles; tc += kJTile) {
    // every thread tests one tile of this chunk: skip it when it cannot hold a listed
    // column of any of the CTA's rows (class S: |c_i - c_j| <= diam_i + diam_j; class N:
    // |c_i - c_j| < eta diam_j)
    {
      const int tt = tc + threadIdx.x;
      bool keep = false;
      if (tt < a.n_tiles) {
        const TileBox b = a.tbox[tt];
        float g2 = 0.f;
        for (int d = 0; d < 3; ++d) {
          const float gap = fmaxf(0.f, fmaxf(s_rb[d] - b.hi[d], b.lo[d] + s_rb[3 + d]));
          g2 += gap * gap;
        }
        const float reach = (b.reach + s_rb[6]) * 1.01f + s_rb[7];
        keep = g2 <= reach * reach;
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      __shared__ int s_wc[kWarps];
      if (lane == 0) s_wc[warp] = __popc(m);
      __syncthreads();
      int base = 0;
      for (int w = 0; w < warp; ++w) base += s_wc[w];
      if (keep) s_live[base + __popc(m & ((1u << lane) - 1u))] = tt;
      if (threadIdx.x == kWarps * 32 - 1) s_nlive = base + __popc(m);
      __syncthreads();
    }
    const int nlive = s_nlive;
    for (int li = 0; li < nlive; ++li) {
      const int64_t j0 = (int64_t)s_live[li] * kJTile;
      __syncthreads();
      for (int t = threadIdx.x; t < kJTile; t += blockDim.x) {
        int64_t j = j0 + t;
        if (j < nt) {
          s_cx[t] = a.cen[j];
          s_cy[t] = a.cen[nt + j];
          s_cz[t] = a.cen[2 * nt + j];
          s_thr[t] = __dmul_rn(a.eta, a.diam[j]);
          s_f[0][t] = (float)s_cx[t];
          s_f[1][t] = (float)s_cy[t];
          s_f[2][t] = (float)s_cz[t];
          s_f[3][t] = (float)s_thr[t];
          s_f[4][t] = (float)a.diam[j];
          s_v[0][t] = a.tri[j];
          s_v[1][t] = a.tri[nt + j];
          s_v[2][t] = a.tri[2 * nt + j];
        }
      }
      __syncthreads();
      const int jn = (int)nat::min64(kJTile, nt - j0);
      for (int jj = 0; jj < jn; jj += 32) {
        const int t = jj + lane;
        const bool in = t < jn;
        const int64_t j = j0 + t;
        float ofx = 3e30f, ofy = 3e30f, ofz = 3e30f, ofth = 0.f, ofd = 0.f;
        if (in) {
          ofx = s_f[0][t];
          ofy = s_f[1][t];
          ofz = s_f[2][t];
          ofth = s_f[3][t];
          ofd = s_f[4][t];
        }
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
          if (!live[q]) continue;  // warp-uniform
          // Conservative fp32 reject: a listed pair has |c_i - c_j| < eta diam_j (class N)
          // or shares a vertex, which implies |c_i - c_j| <= 2/3 (diam_i + diam_j) (class S).
          const float ex = fx[q] - ofx, ey = fy[q] - ofy, ez = fz[q] - ofz;
          const float d2 = ex * ex + ey * ey + ez * ez;
          const float reach = fmaxf(ofth, fd[q] + ofd) * 1.001f + 1e-30f;
          bool hit = false, shares = false;
          if (in && d2 <= reach * reach && j != gi[q]) {
            const int32_t u0 = s_v[0][t], u1 = s_v[1][t], u2 = s_v[2][t];
            shares = (u0 == va[q] || u0 == vb[q] || u0 == vc[q] || u1 == va[q] || u1 == vb[q] ||
                      u1 == vc[q] || u2 == va[q] || u2 == vb[q] || u2 == vc[q]);
            // the exact predicate (reading R-near): fp64, round-to-nearest, no contraction
            double dx = __dsub_rn(s_rc[warp][q][0], s_cx[t]), dy = __dsub_rn(s_rc[warp][q][1], s_cy[t]),
                   dz = __dsub_rn(s_rc[warp][q][2], s_cz[t]);
            double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                               __dmul_rn(dz, dz)));
            hit = shares || dist < s_thr[t];
          }
          unsigned m = __ballot_sync(0xffffffffu, hit);
          if (kBuild) {
            if (hit) {
              int64_t o = pos[q] + __popc(m & ((1u << lane) - 1u));
              a.col[o] = (int32_t)j;
              a.cls[o] = shares ? 1 : 2;
            }
          }
          pos[q] += __popc(m);
        }
      }
    }
    __syncthreads();  // s_live / s_nlive are rewritten by the next chunk
  }
  if (!kBuild && lane == 0) {
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q)
      if (live[q]) a.counts[r0 + q + 1] = pos[q];
  }
}

// Exclusive scan in place over row_ptr[0..rows] (row_ptr[0] = 0, counts in [1..rows]).
// One CTA, fixed segmentation -> deterministic.
__global__ void __launch_bounds__(1024) scan_kernel(int64_t* rp, int64_t rows) {
  __shared__ int64_t sh[33];
  const int t = threadIdx.x;
  const int64_t per = (rows + 1023) / 1024;
  const int64_t b = 1 + t * per, e = nat::min64(rows + 1, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += rp[i];
  int64_t acc = nat::block_exscan_1024(s, sh, nullptr);
  for (int64_t i = b; i < e; ++i) {
    acc += rp[i];
    rp[i] = acc;
  }
  if (t == 0) rp[0] = 0;
}

nat_status check_args(const nat_mesh* mesh, const nat_geom* geom, int64_t row_begin, int64_t row_end) {
  NAT_REQUIRE(mesh && geom, "mesh and geom must be non-null");
  NAT_REQUIRE(geom->n_tri == mesh->n_tri && mesh->n_tri >= 1, "inconsistent n_tri");
  NAT_REQUIRE(mesh->n_tri < (1LL << 31), "n_tri must fit int32");
  NAT_REQUIRE(0 <= row_begin && row_begin < row_end && row_end <= mesh->n_tri,
              "row range [%lld, %lld) outside [0, %lld]", (long long)row_begin, (long long)row_end,
              (long long)mesh->n_tri);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->centroid);
  NAT_REQUIRE_DEV(geom->diam);
  return NAT_OK;
}

double eta_of(const nat_quad_opts* o) { return (o && o->near_eta > 0) ? o->near_eta : 4.0; }

int n_tiles_of(int64_t nt) { return (int)((nt + kJTile - 1) / kJTile); }

// tile boxes into the workspace (shared by the count and build passes)
nat_status prep_tiles(const nat_mesh* mesh, const nat_geom* geom, double eta, void* ws, size_t ws_bytes,
                      NearArgs& a, cudaStream_t s) {
  const int nt_tiles = n_tiles_of(mesh->n_tri);
  const size_t need = sizeof(TileBox) * (size_t)nt_tiles;
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  NAT_REQUIRE_DEV(ws);
  TileBox* tb = static_cast<TileBox*>(ws);
  tile_box_kernel<<<nt_tiles, kJTile, 0, s>>>(mesh->n_tri, geom->centroid, geom->diam, eta, tb);
  NAT_LAUNCH_CHECK();
  a.tbox = tb;
  a.n_tiles = nt_tiles;
  return NAT_OK;
}

}  // namespace

extern "C" size_t nat_bem_near_workspace(int64_t n_tri) {
  return n_tri > 0 ? sizeof(TileBox) * (size_t)n_tiles_of(n_tri) : 0;
}

extern "C" nat_status nat_bem_near_count(const nat_mesh* mesh, const nat_geom* geom,
                                         const nat_quad_opts* opts, int64_t row_begin,
                                         int64_t row_end, int64_t* row_ptr, int64_t* nnz, void* ws,
                                         size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = check_args(mesh, geom, row_begin, row_end);
  if (st != NAT_OK) return st;
  NAT_REQUIRE(nnz, "nnz must be a host pointer");
  NAT_REQUIRE_DEV(row_ptr);
  cudaStream_t s = (cudaStream_t)stream;
  NearArgs a{};
  a.nt = mesh->n_tri;
  a.row_begin = row_begin;
  a.rows = row_end - row_begin;
  a.tri = mesh->tri;
  a.cen = geom->centroid;
  a.diam = geom->diam;
  a.eta = eta_of(opts);
  a.counts = row_ptr;
  st = prep_tiles(mesh, geom, a.eta, ws, ws_bytes, a, s);
  if (st != NAT_OK) return st;
  unsigned grid = (unsigned)((a.rows + kRowsPerCta - 1) / kRowsPerCta);
  near_kernel<false><<<grid, kWarps * 32, 0, s>>>(a);
  scan_kernel<<<1, 1024, 0, s>>>(row_ptr, a.rows);
  NAT_LAUNCH_CHECK();
  NAT_CUDA_TRY(cudaMemcpyAsync(nnz, row_ptr + a.rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  return NAT_OK;
}

extern "C" nat_status nat_bem_near_build(const nat_mesh* mesh, const nat_geom* geom,
                                         const nat_quad_opts* opts, int64_t row_begin,
                                         int64_t row_end, const int64_t* row_ptr, int32_t* col,
                                         uint8_t* cls, void* ws, size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = check_args(mesh, geom, row_begin, row_end);
  if (st != NAT_OK) return st;
  NAT_REQUIRE_DEV(row_ptr);
  NAT_REQUIRE_DEV(col);
  NAT_REQUIRE_DEV(cls);
  NearArgs a{};
  a.nt = mesh->n_tri;
  a.row_begin = row_begin;
  a.rows = row_end - row_begin;
  a.tri = mesh->tri;
  a.cen = geom->centroid;
  a.diam = geom->diam;
  a.eta = eta_of(opts);
  a.row_ptr = row_ptr;
  a.col = col;
  a.cls = cls;
  // the tile boxes are recomputed (cheap), so build does not depend on count's workspace
  st = prep_tiles(mesh, geom, a.eta, ws, ws_bytes, a, (cudaStream_t)stream);
  if (st != NAT_OK) return st;
  unsigned grid = (unsigned)((a.rows + kRowsPerCta - 1) / kRowsPerCta);
  near_kernel<true><<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(a);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
