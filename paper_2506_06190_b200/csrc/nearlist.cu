// Row a2 — near list for the dense BEM ("integrations involving adjacent or
// identical elements"; reading R-near).
//
// For row i (global index) and source triangle j != i:
//   class 1 (S): T_j shares a vertex index with T_i,
//   class 2 (N): otherwise, if sqrt((dx*dx + dy*dy) + dz*dz) < eta*diam_j, d = c_i - c_j,
// evaluated in fp64 with explicit round-to-nearest intrinsics (no FMA contraction), so
// the integer result is identical to the oracle's.  CSR, columns ascending.
//
// Kernel: CTA = 8 warps x 4 rows each; source triangles are staged in shared-memory
// tiles of 256 shared by the CTA's 32 rows; each warp scans its rows' candidates 32 at
// a time and compacts hits with __ballot_sync (ascending order is preserved).
#include "nat_internal.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kRowsPerWarp = 4;
constexpr int kRowsPerCta = kWarps * kRowsPerWarp;
constexpr int kJTile = 256;

struct NearArgs {
  int64_t nt, row_begin, rows;
  const int32_t* tri;
  const double* cen;
  const double* diam;
  double eta;
  const int64_t* row_ptr;  // build pass: offsets (relative to row_begin)
  int64_t* counts;         // count pass: counts[r + 1]
  int32_t* col;
  uint8_t* cls;
};

template <bool kBuild>
__global__ void __launch_bounds__(kWarps * 32) near_kernel(NearArgs a) {
  __shared__ double s_cx[kJTile], s_cy[kJTile], s_cz[kJTile], s_thr[kJTile];
  __shared__ float s_f[5][kJTile];  // fp32 centroid, eta*diam, diam: conservative prefilter
  __shared__ int32_t s_v[3][kJTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta + warp * kRowsPerWarp;
  const int64_t nt = a.nt;

  // the rows' fp64 centroids live in shared memory (used only by the exact test, rarely)
  __shared__ double s_rc[kWarps][kRowsPerWarp][3];
  __shared__ float s_rd[kWarps][kRowsPerWarp];
  __shared__ float s_rb[8];            // rows: min xyz, -max xyz, max diam, fp32 margin
  __shared__ float s_tb[kWarps][7];    // tile reduction scratch
  __shared__ int s_skip;
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

  for (int64_t j0 = 0; j0 < nt; j0 += kJTile) {
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
    // tile bounding box + reach (fp32, conservative): skip the whole tile when it cannot
    // hold a listed column of any of this CTA's rows (uniform branch)
    {
      const int t = threadIdx.x;
      const bool ok = j0 + t < nt;
      float v[7] = {ok ? s_f[0][t] : 3e30f, ok ? s_f[1][t] : 3e30f, ok ? s_f[2][t] : 3e30f,
                    ok ? -s_f[0][t] : 3e30f, ok ? -s_f[1][t] : 3e30f, ok ? -s_f[2][t] : 3e30f,
                    ok ? -fmaxf(s_f[3][t], s_f[4][t]) : 0.f};
      // v[6] holds -max(eta diam, diam); min-reductions throughout
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < 7; ++c) v[c] = fminf(v[c], __shfl_xor_sync(0xffffffffu, v[c], o));
      if (lane == 0)
#pragma unroll
        for (int c = 0; c < 7; ++c) s_tb[warp][c] = v[c];
      __syncthreads();
      if (threadIdx.x == 0) {
        float b[7];
        for (int c = 0; c < 7; ++c) {
          b[c] = s_tb[0][c];
          for (int w = 1; w < kWarps; ++w) b[c] = fminf(b[c], s_tb[w][c]);
        }
        float g2 = 0.f;
        for (int d = 0; d < 3; ++d) {
          // rows: [s_rb[d], -s_rb[3+d]], tile: [b[d], -b[3+d]]
          const float gap = fmaxf(0.f, fmaxf(s_rb[d] + b[3 + d], b[d] + s_rb[3 + d]));
          g2 += gap * gap;
        }
        const float reach = fmaxf(-b[6], s_rb[6] + (-b[6])) * 1.01f + s_rb[7];
        s_skip = g2 > reach * reach;
      }
      __syncthreads();
      if (s_skip) continue;
    }
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
        // Conservative fp32 reject: a listed pair has |c_i - c_j| < eta diam_j (class N) or
        // shares a vertex, which implies |c_i - c_j| <= 2/3 (diam_i + diam_j) (class S).
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
  if (!kBuild && lane == 0) {
#pragma unroll
    for (int q = 0; q < kRowsPerWarp; ++q)
      if (live[q]) a.counts[r0 + q + 1] = pos[q];
  }
}

// Exclusive scan in place over row_ptr[0..rows] (row_ptr[0] = 0, counts in [1..rows]).
// One CTA, fixed segmentation -> deterministic.
__global__ void __launch_bounds__(1024) scan_kernel(int64_t* rp, int64_t rows) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (rows + 1023) / 1024;
  const int64_t b = 1 + t * per, e = nat::min64(rows + 1, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += rp[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int q = 0; q < 1024; ++q) {
      int64_t v = part[q];
      part[q] = acc;
      acc += v;
    }
  }
  __syncthreads();
  int64_t acc = part[t];
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

}  // namespace

extern "C" nat_status nat_bem_near_count(const nat_mesh* mesh, const nat_geom* geom,
                                         const nat_quad_opts* opts, int64_t row_begin,
                                         int64_t row_end, int64_t* row_ptr, int64_t* nnz,
                                         nat_stream_t stream) {
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
                                         uint8_t* cls, nat_stream_t stream) {
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
  unsigned grid = (unsigned)((a.rows + kRowsPerCta - 1) / kRowsPerCta);
  near_kernel<true><<<grid, kWarps * 32, 0, (cudaStream_t)stream>>>(a);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
