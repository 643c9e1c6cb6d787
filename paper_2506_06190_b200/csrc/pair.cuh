// Device-side Helmholtz pair evaluation helpers, fp32 and fp64.
#pragma once
#include <cuda_runtime.h>

namespace nat {

template <typename T>
struct C2 {
  T x, y;
};

__device__ __forceinline__ float pair_rsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double pair_rsqrt(double x) { return rsqrt(x); }

__device__ __forceinline__ void pair_sincos(float x, float* s, float* c) { __sincosf(x, s, c); }
__device__ __forceinline__ void pair_sincos(double x, double* s, double* c) { sincos(x, s, c); }

// Accumulates, for target x and source point y (d = y - x) with weight w (already
// divided by 4 pi) and source normal n:
//   V += w G-part = w rho e^{ikr}                         (single layer, 4 pi G = e^{ikr}/r)
//   K += w dn rho^3 (ikr - 1) e^{ikr}                     (double layer, 4 pi dG/dn_y)
template <typename R>
__device__ __forceinline__ void pair_accumulate(R dx, R dy, R dz, R nx, R ny, R nz, R w, R k,
                                                R& Vr, R& Vi, R& Kr, R& Ki) {
  const R r2 = dx * dx + dy * dy + dz * dz;
  const R dn = dx * nx + dy * ny + dz * nz;
  const R rho = pair_rsqrt(r2);
  const R rr = r2 * rho;
  const R kr = k * rr;
  R s, c;
  pair_sincos(kr, &s, &c);
  const R t = w * rho;
  Vr += t * c;
  Vi += t * s;
  const R u = t * dn * (rho * rho);
  Kr += u * (-c - kr * s);
  Ki += u * (kr * c - s);
}

// Burton-Miller pair (Eq. BM; reading R-bm): with the target normal n_x also
//   K' += w (-d.n_x) rho^3 (ikr - 1) e^{ikr}                         (4 pi dG/dn_x)
//   W  += w rho^3 [-(d.n_x)(d.n_y) rho^2 (3 - 3ikr - k^2 r^2) - (n_x.n_y)(ikr - 1)] e^{ikr}
//                                                                     (4 pi d2G/dn_x dn_y)
template <typename R>
__device__ __forceinline__ void pair_accumulate_bm(R dx, R dy, R dz, R nx, R ny, R nz, R mx, R my, R mz, R w,
                                                   R k, C2<R>& V, C2<R>& K, C2<R>& Kp, C2<R>& W) {
  const R r2 = dx * dx + dy * dy + dz * dz;
  const R dn = dx * nx + dy * ny + dz * nz;   // d . n_y
  const R dm = dx * mx + dy * my + dz * mz;   // d . n_x
  const R nn = nx * mx + ny * my + nz * mz;   // n_x . n_y
  const R rho = pair_rsqrt(r2);
  const R rr = r2 * rho;
  const R kr = k * rr;
  R s, c;
  pair_sincos(kr, &s, &c);
  const R t = w * rho;
  V.x += t * c;
  V.y += t * s;
  const R rho2 = rho * rho;
  const R er = -c - kr * s, ei = kr * c - s;  // (ikr - 1) e^{ikr}
  const R uy = t * dn * rho2, ux = -t * dm * rho2;
  K.x += uy * er;
  K.y += uy * ei;
  Kp.x += ux * er;
  Kp.y += ux * ei;
  const R q1 = -dn * dm * rho2;
  const R br = q1 * (R(3) - kr * kr) + nn, bi = -kr * (R(3) * q1 + nn);  // bracket
  const R tw = t * rho2;
  W.x += tw * (br * c - bi * s);
  W.y += tw * (br * s + bi * c);
}

}  // namespace nat

namespace nat {
// Squared distance in fp32 exactly as the radiation / MC kernels form it.  The MC
// near-pair list uses the same function so that the pairs the fp32 kernel skips are
// exactly the pairs evaluated in fp64.
__device__ __forceinline__ float pair_r2_f32(float dx, float dy, float dz) {
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}
}  // namespace nat
