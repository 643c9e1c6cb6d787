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
// fp64 sin/cos for the pair kernels.  libm's sincos materialises its ~20 fp64 constants
// with UMOV/IMAD pairs at every call (DFMA takes no 64-bit immediate; ~50 of the ~117
// instructions per fp64 pair in SASS, issue-bound kernels); here the constants live in
// the constant bank, which DFMA reads directly.  Quadrant q = rint(2x/pi) by the
// 1.5 * 2^52 shift, 3-term Cody-Waite reduction with FMA (accurate for |x| < 2^20 pi/2
// ~ 1.6e6, i.e. up to 2.6e5 wavelengths across a mesh; beyond that libm), fdlibm
// __kernel_sin / __kernel_cos polynomials on |r| <= pi/4.
__constant__ double kPairTrig[17] = {
    0.63661977236758134308,                       // 2/pi
    6755399441055744.0,                           // 1.5 * 2^52
    1.5707963267948966e+00, 6.123233995736766e-17, -1.4973849048591698e-33,  // pi/2 (3 parts)
    1.58969099521155010221e-10, -2.50507602534068634195e-08, 2.75573137070700676789e-06,
    -1.98412698298579493134e-04, 8.33333333332248946124e-03, -1.66666666666666324348e-01,  // sin
    -1.13596475577881948265e-11, 2.08757232129817482790e-09, -2.75573143513906633035e-07,
    2.48015872894767294178e-05, -1.38888888888741095749e-03, 4.16666666666666019037e-02};  // cos

static __device__ __noinline__ void pair_sincos_libm(double x, double* s, double* c) { sincos(x, s, c); }

__device__ __forceinline__ void pair_sincos(double x, double* s, double* c) {
  if (!(fabs(x) < 1.6e6)) {
    pair_sincos_libm(x, s, c);
    return;
  }
  const double* K = kPairTrig;
  const double t = fma(x, K[0], K[1]);
  const int qi = __double2loint(t);
  const double q = t - K[1];
  double r = fma(-q, K[2], x);
  r = fma(-q, K[3], r);
  r = fma(-q, K[4], r);
  const double z = r * r;
  double ps = fma(z, K[5], K[6]);
  ps = fma(z, ps, K[7]);
  ps = fma(z, ps, K[8]);
  ps = fma(z, ps, K[9]);
  ps = fma(z, ps, K[10]);
  const double sr = fma(r * z, ps, r);
  double pc = fma(z, K[11], K[12]);
  pc = fma(z, pc, K[13]);
  pc = fma(z, pc, K[14]);
  pc = fma(z, pc, K[15]);
  pc = fma(z, pc, K[16]);
  const double cr = fma(z * z, pc, fma(-0.5, z, 1.0));
  const double so = (qi & 1) ? cr : sr;
  const double co = (qi & 1) ? sr : cr;
  // quadrant signs by flipping the sign bit (integer pipe, not a DADD)
  *s = __longlong_as_double(__double_as_longlong(so) ^ ((long long)(qi & 2) << 62));
  *c = __longlong_as_double(__double_as_longlong(co) ^ ((long long)((qi + 1) & 2) << 62));
}

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
