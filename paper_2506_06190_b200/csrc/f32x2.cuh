// Packed FP32x2 arithmetic (PTX add/sub/mul/fma .f32x2 -> SASS FADD2/FMUL2/FFMA2,
// sm_100a): two lanes of fp32 work per instruction issue.
#pragma once
#include <cuda_runtime.h>

namespace {
typedef unsigned long long f2r;  // a float2 in a 64-bit register pair
__device__ __forceinline__ f2r f2pack(float lo, float hi) {
  f2r r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2lo(f2r a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  return lo;
}
__device__ __forceinline__ float f2hi(f2r a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  return hi;
}
__device__ __forceinline__ f2r f2add(f2r a, f2r b) {
  f2r r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2r f2sub(f2r a, f2r b) {
  f2r r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2r f2mul(f2r a, f2r b) {
  f2r r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2r f2fma(f2r a, f2r b, f2r c) {
  f2r r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

}  // namespace
