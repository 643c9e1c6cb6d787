// Microbenchmark of the issue/pipe rates that bound the pair kernels on this B200:
// scalar FFMA, packed FFMA2 (fma.rn.f32x2), MUFU (ex2.approx: no pre-multiply) and
// sin.approx (FMUL.RZ + MUFU.SIN).  8 independent chains per thread, full grid.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, 0.5f);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a) {
  unsigned long long x[8], av, bv;
  float lo = a, hi = a;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(lo), "f"(hi));
  float h = 0.5f;
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(h), "f"(h));
  for (int i = 0; i < 8; ++i) {
    float v = threadIdx.x + i;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(v), "f"(v));
  }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float l2, h2;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(l2), "=f"(h2) : "l"(x[i]));
    s += l2 + h2;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ex2(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_sin(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __sinf(x[i]);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(float* out, float a) {
  double x[8];
  const double ad = a;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], ad, 0.5);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

__global__ void k_rsq(float* out, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + i) * 1e-3f + 1.f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
double run(K k, float* out, int blocks, int threads) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<blocks, threads>>>(out, 1.0001f);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, 1.0001f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5 * 1e-3;
}

int main() {
  int dev = 0, sms = 0, mhz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
  const int threads = 256, blocks = sms * 8;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  const double ops = (double)blocks * threads * kIters * 8;  // thread-level ops per launch
  double t;
  t = run(k_ffma, out, blocks, threads);
  printf("FFMA  : %.3e lane-ops/s = %.1f per SM per clk (at %d MHz)\n", ops / t, ops / t / sms / (mhz * 1e3), mhz / 1000);
  t = run(k_ffma2, out, blocks, threads);
  printf("FFMA2 : %.3e instr-lanes/s (x2 fp32 ops) = %.1f fp32 ops per SM per clk\n", ops / t, 2 * ops / t / sms / (mhz * 1e3));
  t = run(k_ex2, out, blocks, threads);
  printf("MUFU.EX2: %.3e lane-ops/s = %.1f per SM per clk\n", ops / t, ops / t / sms / (mhz * 1e3));
  t = run(k_sin, out, blocks, threads);
  printf("__sinf (FMUL.RZ+MUFU.SIN): %.3e /s = %.1f per SM per clk\n", ops / t, ops / t / sms / (mhz * 1e3));
  t = run(k_rsq, out, blocks, threads);
  printf("MUFU.RSQ: %.3e lane-ops/s = %.1f per SM per clk\n", ops / t, ops / t / sms / (mhz * 1e3));
  t = run(k_dfma, out, blocks, threads);
  printf("DFMA  : %.3e lane-ops/s = %.1f per SM per clk (FP64 pipe)\n", ops / t, ops / t / sms / (mhz * 1e3));
  return 0;
}
