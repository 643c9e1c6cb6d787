// Internal helpers of libnat (not part of the ABI).
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/nat.h"

namespace nat {

void set_error(const char* fmt, ...);
nat_status fail(nat_status st, const char* fmt, ...);
bool is_device_ptr(const void* p);

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kInv4Pi = 0.0795774715459476678844418816862571810;
constexpr int kNumSMs = 148;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// NVTX range around every nat_* entry point (named after the call; header-only NVTX v3,
// a no-op unless a tool such as nsys / ncu --nvtx is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define NAT_TRACE() ::nat::NvtxRange nat_nvtx_range_(__func__)

// Carves sub-buffers out of a caller workspace (256-byte aligned pieces).
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t bytes() const { return align_up(off, 256); }
};

int device_sm_count();

// Kernel timer (nat_kernel_timer_*, diagnostics): events around the main kernel of a
// category on the launching stream; `pairs` = algorithmic pair-evaluations of the launch;
// `skip` (optional device word) marks launches that returned at once (not counted).
enum { kTimerMcOp = 0, kTimerMcRhs = 1, kTimerRadiate = 2, kTimerFar = 3, kTimerNfGemm = 4, kTimerCats = 5 };
bool ktimer_on();
void ktimer_begin(int cat, cudaStream_t s);
// n_modes: wavenumbers evaluated per pair by the launch (roofline bucket; 0 = none)
void ktimer_end(int cat, cudaStream_t s, double pairs, const unsigned long long* skip, int n_modes = 0);

// Exclusive scan of one int64 per thread over a 1024-thread block (warp shuffles, exact);
// sh: 33 int64 of shared memory; *total (optional) receives the block sum.
__device__ __forceinline__ int64_t block_exscan_1024(int64_t v, int64_t* sh, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int64_t w = sh[lane];
    int64_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    sh[lane] = z - w;
    if (lane == 31) sh[32] = z;
  }
  __syncthreads();
  const int64_t r = sh[warp] + x - v;
  if (total) *total = sh[32];
  return r;
}

}  // namespace nat

#define NAT_CUDA_TRY(expr)                                                                   \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return nat::fail(NAT_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),        \
                       __FILE__, __LINE__);                                                  \
  } while (0)

#define NAT_LAUNCH_CHECK()                                                                   \
  do {                                                                                       \
    cudaError_t _e = cudaGetLastError();                                                     \
    if (_e != cudaSuccess)                                                                   \
      return nat::fail(NAT_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(_e),   \
                       __FILE__, __LINE__);                                                  \
  } while (0)

#define NAT_REQUIRE(cond, ...)                                                               \
  do {                                                                                       \
    if (!(cond)) return nat::fail(NAT_ERR_INVALID_ARG, __VA_ARGS__);                          \
  } while (0)

#define NAT_REQUIRE_DEV(ptr)                                                                 \
  NAT_REQUIRE(nat::is_device_ptr(ptr), "%s must be a device pointer", #ptr)

namespace nat {
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
}  // namespace nat
