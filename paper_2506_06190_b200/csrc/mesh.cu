// Row a1 — mesh preparation (reading R-geom) and
// row a12 — listener shell grid (reading R-listen).
//
// Every fp64 operation that feeds an integer decision downstream (near list, MC
// triangle choice, MC sample position) is written with explicit round-to-nearest
// intrinsics (__dadd_rn, __dmul_rn, ...) so nvcc cannot contract it into an FMA:
// the results are bit-identical to any IEEE implementation of the same formula.
#include "nat_internal.cuh"
#include "philox.cuh"

namespace {

struct PrepScalars {
  double total_area, cx, cy, cz, volume, radius;
  long long bad_tri;  // min index of a zero-area triangle, or LLONG_MAX
};

__device__ __forceinline__ double dnorm_rn(double x, double y, double z) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

__global__ void tri_geom_kernel(int64_t nv, int64_t nt, const double* __restrict__ vx,
                                const int32_t* __restrict__ tri, double* __restrict__ cen,
                                double* __restrict__ nrm, double* __restrict__ area,
                                double* __restrict__ diam, double* __restrict__ vol_term,
                                PrepScalars* sc) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const double* X = vx;
  const double* Y = vx + nv;
  const double* Z = vx + 2 * nv;
  int a = tri[t], b = tri[nt + t], c = tri[2 * nt + t];
  double x1 = X[a], y1 = Y[a], z1 = Z[a];
  double x2 = X[b], y2 = Y[b], z2 = Z[b];
  double x3 = X[c], y3 = Y[c], z3 = Z[c];
  double ax = __dsub_rn(x2, x1), ay = __dsub_rn(y2, y1), az = __dsub_rn(z2, z1);
  double bx = __dsub_rn(x3, x1), by = __dsub_rn(y3, y1), bz = __dsub_rn(z3, z1);
  double ex = __dsub_rn(__dmul_rn(ay, bz), __dmul_rn(az, by));
  double ey = __dsub_rn(__dmul_rn(az, bx), __dmul_rn(ax, bz));
  double ez = __dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx));
  double en = dnorm_rn(ex, ey, ez);
  if (!(en > 0.0)) atomicMin(&sc->bad_tri, (long long)t);
  area[t] = __dmul_rn(0.5, en);
  nrm[t] = __ddiv_rn(ex, en);
  nrm[nt + t] = __ddiv_rn(ey, en);
  nrm[2 * nt + t] = __ddiv_rn(ez, en);
  cen[t] = __ddiv_rn(__dadd_rn(__dadd_rn(x1, x2), x3), 3.0);
  cen[nt + t] = __ddiv_rn(__dadd_rn(__dadd_rn(y1, y2), y3), 3.0);
  cen[2 * nt + t] = __ddiv_rn(__dadd_rn(__dadd_rn(z1, z2), z3), 3.0);
  double l12 = dnorm_rn(__dsub_rn(x2, x1), __dsub_rn(y2, y1), __dsub_rn(z2, z1));
  double l23 = dnorm_rn(__dsub_rn(x3, x2), __dsub_rn(y3, y2), __dsub_rn(z3, z2));
  double l31 = dnorm_rn(__dsub_rn(x1, x3), __dsub_rn(y1, y3), __dsub_rn(z1, z3));
  diam[t] = fmax(fmax(l12, l23), l31);
  // v1 . (v2 x v3) for the signed volume (order of the final sum is irrelevant)
  vol_term[t] = x1 * (y2 * z3 - z2 * y3) + y1 * (z2 * x3 - x2 * z3) + z1 * (x2 * y3 - y2 * x3);
}

// Sequential prefix sum, exactly the left-to-right order of the definition.
// The block stages chunks of the areas in shared memory (coalesced), thread 0 runs the
// dependent fp64 chain out of shared memory, the block writes the chunk back.
constexpr int kCdfChunk = 4096;
__global__ void __launch_bounds__(1024) cdf_kernel(int64_t nt, const double* __restrict__ area,
                                                   double* __restrict__ cdf) {
  __shared__ double buf[kCdfChunk];
  double s = 0.0;
  for (int64_t c0 = 0; c0 < nt; c0 += kCdfChunk) {
    const int len = (int)nat::min64(kCdfChunk, nt - c0);
    for (int t = threadIdx.x; t < len; t += blockDim.x) buf[t] = area[c0 + t];
    __syncthreads();
    if (threadIdx.x == 0) {
      // 8 loads, 8 dependent adds, 8 stores: only the fp64 add latency stays serial
      // (adding the 0.0 padding past `len` leaves s unchanged)
      for (int t = 0; t < len; t += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = t + u < len ? buf[t + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s = __dadd_rn(s, v[u]);
          v[u] = s;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t + u < len) buf[t + u] = v[u];
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < len; t += blockDim.x) cdf[c0 + t] = buf[t];
    __syncthreads();
  }
}

constexpr int RB = 1024;

// One block.  centre = sum_t A_t c_t / |Gamma| with the sums taken sequentially, left to
// right, every product and sum rounded (no FMA): the definition's order, so the result is
// bit-identical with the oracle (which accumulates the same products with np.cumsum).
// The block stages RB products per component in shared memory; lane 0 of warps 0..2 runs
// the dependent chain of component 0..2 (8 loads, then 8 adds, per step).  The signed
// volume only decides the orientation check (tree sum; any order).
__global__ void __launch_bounds__(RB) centre_kernel(int64_t nt, const double* __restrict__ area,
                                                    const double* __restrict__ cen,
                                                    const double* __restrict__ vol_term,
                                                    const double* __restrict__ cdf, PrepScalars* sc) {
  __shared__ double prod[3][RB];
  __shared__ double red[RB];
  double acc = 0.0, vol = 0.0;  // acc: the chain of component (warp id) in lane 0 of warps 0..2
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t c0 = 0; c0 < nt; c0 += RB) {
    const int len = (int)nat::min64(RB, nt - c0);
    if (threadIdx.x < len) {
      const int64_t t = c0 + threadIdx.x;
      const double a = area[t];
      prod[0][threadIdx.x] = __dmul_rn(a, cen[t]);
      prod[1][threadIdx.x] = __dmul_rn(a, cen[nt + t]);
      prod[2][threadIdx.x] = __dmul_rn(a, cen[2 * nt + t]);
      vol += vol_term[t];
    }
    __syncthreads();
    if (warp < 3 && lane == 0) {
      const double* pd = prod[warp];
      for (int t = 0; t < len; t += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = t + u < len ? pd[t + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t + u < len) acc = __dadd_rn(acc, v[u]);
      }
    }
    __syncthreads();
  }
  red[threadIdx.x] = vol;
  __syncthreads();
  for (int w = RB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double tot = cdf[nt - 1];
  if (warp < 3 && lane == 0) {
    const double c = __ddiv_rn(acc, tot);
    if (warp == 0) sc->cx = c;
    if (warp == 1) sc->cy = c;
    if (warp == 2) sc->cz = c;
  }
  if (threadIdx.x == 0) {
    sc->total_area = tot;
    sc->volume = red[0] / 6.0;
  }
}

// R = max over vertices of |v - centre|, each distance sqrt((dx dx + dy dy) + dz dz) with
// every operation rounded (the oracle's order); max is order-free.
__global__ void __launch_bounds__(RB) radius_kernel(int64_t nv, const double* __restrict__ vx,
                                                    PrepScalars* sc) {
  __shared__ double red[RB];
  double cx = sc->cx, cy = sc->cy, cz = sc->cz, m = 0.0;
  for (int64_t v = threadIdx.x; v < nv; v += RB) {
    const double dx = __dsub_rn(vx[v], cx), dy = __dsub_rn(vx[nv + v], cy), dz = __dsub_rn(vx[2 * nv + v], cz);
    m = fmax(m, dnorm_rn(dx, dy, dz));
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int w = RB / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) sc->radius = red[0];
}

__global__ void init_scalars(PrepScalars* sc) {
  sc->total_area = sc->cx = sc->cy = sc->cz = sc->volume = sc->radius = 0.0;
  sc->bad_tri = 0x7fffffffffffffffLL;
}

__global__ void listener_grid_kernel(double cx, double cy, double cz, double R, int nth, int nph,
                                     int nr, double r_lo, double r_hi, double* __restrict__ out) {
  int64_t n = (int64_t)nth * nph * nr;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int u = (int)(i % nth);
  int v = (int)((i / nth) % nph);
  int w = (int)(i / ((int64_t)nth * nph));
  const double pi = nat::kPi;
  double th = -pi + (u + 0.5) * 2.0 * pi / nth;
  double ph = (v + 0.5) * pi / nph;
  double r = R * (r_lo + (r_hi - r_lo) * (w + 0.5) / nr);
  double st, ct, sp, cp;
  sincos(th, &st, &ct);
  sincos(ph, &sp, &cp);
  out[i] = cx + r * (sp * ct);
  out[n + i] = cy + r * (sp * st);
  out[2 * n + i] = cz + r * cp;
}

// Reading R-listen-rand: point t of a random shell, uniform in volume
// (SPEC's design note to P:166): Philox counter (t, 1, stream_lo, stream_hi), key = seed,
// u_a = (o_a + 1/2) 2^-32;  cos(phi) = 1 - 2 u0, sin(phi) = 2 sqrt(u0 (1 - u0)),
// theta = -pi + 2 pi u1,  r = R cbrt(r_lo^3 + u2 (r_hi^3 - r_lo^3)).
__global__ void listener_random_kernel(double cx, double cy, double cz, double R, int64_t n, double r_lo,
                                       double r_hi, uint64_t seed, uint64_t stream_id, double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  uint32_t c0 = (uint32_t)t, c1 = 1u, c2 = (uint32_t)stream_id, c3 = (uint32_t)(stream_id >> 32);
  nat::philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double two32 = 2.3283064365386963e-10;  // 2^-32
  const double u0 = ((double)c0 + 0.5) * two32, u1 = ((double)c1 + 0.5) * two32, u2 = ((double)c2 + 0.5) * two32;
  const double cp = 1.0 - 2.0 * u0, sp = 2.0 * sqrt(u0 * (1.0 - u0));
  double st, ct;
  sincos(-nat::kPi + 2.0 * nat::kPi * u1, &st, &ct);
  const double lo3 = r_lo * r_lo * r_lo, hi3 = r_hi * r_hi * r_hi;
  const double r = R * cbrt(lo3 + u2 * (hi3 - lo3));
  out[t] = cx + r * (sp * ct);
  out[n + t] = cy + r * (sp * st);
  out[2 * n + t] = cz + r * cp;
}

}  // namespace

extern "C" size_t nat_mesh_prepare_workspace(int64_t n_vert, int64_t n_tri) {
  (void)n_vert;
  nat::Carver c(nullptr);
  c.take<PrepScalars>(1);
  c.take<double>(n_tri);
  return c.bytes();
}

extern "C" nat_status nat_mesh_prepare(const nat_mesh* mesh, nat_geom* geom, void* ws,
                                       size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(mesh && geom, "mesh and geom must be non-null");
  NAT_REQUIRE(mesh->n_vert >= 3 && mesh->n_tri >= 1, "need n_vert >= 3 and n_tri >= 1");
  NAT_REQUIRE(geom->n_tri == mesh->n_tri, "geom->n_tri (%lld) != mesh->n_tri (%lld)",
              (long long)geom->n_tri, (long long)mesh->n_tri);
  NAT_REQUIRE_DEV(mesh->vxyz);
  NAT_REQUIRE_DEV(mesh->tri);
  NAT_REQUIRE_DEV(geom->centroid);
  NAT_REQUIRE_DEV(geom->normal);
  NAT_REQUIRE_DEV(geom->area);
  NAT_REQUIRE_DEV(geom->diam);
  NAT_REQUIRE_DEV(geom->area_cdf);
  size_t need = nat_mesh_prepare_workspace(mesh->n_vert, mesh->n_tri);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  NAT_REQUIRE_DEV(ws);
  nat::Carver c(ws);
  PrepScalars* sc = c.take<PrepScalars>(1);
  double* vol = c.take<double>(mesh->n_tri);
  cudaStream_t s = (cudaStream_t)stream;
  int64_t nt = mesh->n_tri;
  init_scalars<<<1, 1, 0, s>>>(sc);
  tri_geom_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(
      mesh->n_vert, nt, mesh->vxyz, mesh->tri, geom->centroid, geom->normal, geom->area, geom->diam,
      vol, sc);
  cdf_kernel<<<1, 1024, 0, s>>>(nt, geom->area, geom->area_cdf);
  centre_kernel<<<1, RB, 0, s>>>(nt, geom->area, geom->centroid, vol, geom->area_cdf, sc);
  radius_kernel<<<1, RB, 0, s>>>(mesh->n_vert, mesh->vxyz, sc);
  NAT_LAUNCH_CHECK();
  PrepScalars h;
  NAT_CUDA_TRY(cudaMemcpyAsync(&h, sc, sizeof h, cudaMemcpyDeviceToHost, s));
  NAT_CUDA_TRY(cudaStreamSynchronize(s));
  if (h.bad_tri != 0x7fffffffffffffffLL)
    return nat::fail(NAT_ERR_SINGULAR, "zero-area triangle %lld", h.bad_tri);
  if (!(h.volume > 0.0))
    return nat::fail(NAT_ERR_SINGULAR, "mesh is not outward-oriented (signed volume %g <= 0)",
                     h.volume);
  geom->total_area = h.total_area;
  geom->center[0] = h.cx;
  geom->center[1] = h.cy;
  geom->center[2] = h.cz;
  geom->bound_radius = h.radius;
  geom->volume = h.volume;
  return NAT_OK;
}

extern "C" nat_status nat_listener_grid(const double* center, double R, int n_theta, int n_phi,
                                        int n_r, double r_lo, double r_hi, double* out,
                                        nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(center, "center must be a host pointer to 3 doubles");
  NAT_REQUIRE(n_theta > 0 && n_phi > 0 && n_r > 0, "grid sizes must be positive");
  NAT_REQUIRE(R > 0 && r_lo > 0 && r_hi >= r_lo, "need R > 0, 0 < r_lo <= r_hi");
  NAT_REQUIRE_DEV(out);
  int64_t n = (int64_t)n_theta * n_phi * n_r;
  listener_grid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      center[0], center[1], center[2], R, n_theta, n_phi, n_r, r_lo, r_hi, out);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

extern "C" nat_status nat_listener_random_shell(const double* center, double R, int64_t n, double r_lo,
                                                double r_hi, uint64_t seed, uint64_t stream_id, double* out,
                                                nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(center, "center must be a host array of 3");
  NAT_REQUIRE(n >= 1, "need n >= 1");
  NAT_REQUIRE(R > 0 && r_lo > 0 && r_hi >= r_lo, "need R > 0, 0 < r_lo <= r_hi");
  NAT_REQUIRE_DEV(out);
  listener_random_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      center[0], center[1], center[2], R, n, r_lo, r_hi, seed, stream_id, out);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}
