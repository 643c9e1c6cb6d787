// NEXT-4 — the NAT neural acoustic transfer field (§3.2-3.3, l.120-162;
// reading R-nf): multi-resolution feature grid G(theta, phi, r) (4 levels,
// 8..64, 4 features, trilinear), NeRF positional encoding of the condition variables
// (2^0..2^5), a 4 x 128 ReLU MLP, MSE loss and Adam — forward and one training step.
//
// B200 design: every layer product (forward, input gradient, weight gradient) runs on the
// 5th-generation tensor cores: `tcgen05.mma.cta_group::1.kind::f16` (bf16 operands, fp32
// accumulators in TMEM), issued by one thread per CTA, operands staged in shared memory in
// the canonical no-swizzle core-matrix layout (K-major or MN-major, so row-major
// activations serve both as [batch][features] and transposed without copies), two smem
// stages with tcgen05.commit -> mbarrier handshakes, TMEM -> registers with tcgen05.ld for
// fused epilogues (bias + ReLU + bf16, ReLU-mask, fp32 split-K partials).  Encoding,
// loss, grid scatter and Adam are elementwise kernels.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "async_copy.cuh"
#include "nat_internal.cuh"

namespace {

using bf16 = __nv_bfloat16;

constexpr int kLevels = 4, kFeat = 4, kBaseRes = 8, kTable = 1 << 19, kPeFreq = 6;
constexpr int kInPad = 64, kHidden = 128, kNHidden = 4, kOutPad = 16;
constexpr int kNLayers = kNHidden + 1;

__host__ __device__ constexpr int level_res(int l) { return kBaseRes << l; }
__host__ __device__ constexpr int64_t level_rows(int l) {  // dense when the lattice fits the table
  return (int64_t)(level_res(l) + 1) * (level_res(l) + 1) * (level_res(l) + 1) <= kTable
             ? (int64_t)(level_res(l) + 1) * (level_res(l) + 1) * (level_res(l) + 1)
             : (int64_t)kTable;
}
__device__ __forceinline__ int64_t vertex_row(int l, int64_t i, int64_t j, int64_t k) {
  const int64_t n = level_res(l) + 1;
  if (n * n * n <= kTable) return i + n * (j + n * k);
  const uint64_t h = ((uint64_t)i * 1ull) ^ ((uint64_t)j * 2654435761ull) ^ ((uint64_t)k * 805459861ull);
  return (int64_t)(h % (uint64_t)kTable);
}

// ---- parameter layout (the oracle's order): grid0..3 [rows][4], then W_q [out][in], b_q ----
struct Layout {
  int64_t grid[kLevels];
  int64_t W[kNLayers], b[kNLayers];
  int in[kNLayers], out[kNLayers];
  int64_t total;
};
Layout layout_of(int n_out) {
  Layout L{};
  int64_t o = 0;
  for (int l = 0; l < kLevels; ++l) {
    L.grid[l] = o;
    o += level_rows(l) * kFeat;
  }
  for (int q = 0; q < kNLayers; ++q) {
    L.in[q] = q == 0 ? kInPad : kHidden;
    L.out[q] = q == kNHidden ? n_out : kHidden;
    L.W[q] = o;
    o += (int64_t)L.in[q] * L.out[q];
    L.b[q] = o;
    o += L.out[q];
  }
  L.total = o;
  return L;
}

// =====================================================================================
// tcgen05 GEMM: C[M x N] = A[M x K] * B[N x K]^T, bf16 operands, fp32 accumulation in TMEM.
// A is K-major (A[m * lda + k]) or MN-major (A[k * lda + m]); likewise B (B[n * ldb + k] or
// B[k * ldb + n]).  One CTA = 128 rows x N (N in {16, 32, 64, 128}), K in chunks of 64.
// =====================================================================================
constexpr int kGM = 128, kBK = 64, kGT = 256;  // 8 warps: warp w reads TMEM lanes 32 (w % 4)

enum Epi : int {
  kEpiBiasReluBf16 = 0,  // Cb = bf16(relu(acc + bias))
  kEpiBiasF32 = 1,       // C = acc + bias        (columns < n_valid)
  kEpiMaskBf16 = 2,      // v = acc * (H > 0): Cb = bf16(v), column sums of v -> colpart[tile][n]
  kEpiF32 = 3,           // C = acc
  kEpiPartial = 4,       // C[split][M][N] = acc  (split-K partial)
};

struct GemmArgs {
  const bf16* A;
  int64_t lda;
  const bf16* B;
  int64_t ldb;
  int64_t M, N, K, k_per_cta;
  int epi, n_valid;
  float* C;
  int64_t ldc;
  bf16* Cb;
  const float* bias;
  int n_bias;       // bias entries (the rest of the tile reads 0)
  const bf16* H;
  int64_t ldh;
  float* colpart;  // kEpiMaskBf16: [gridDim.x][N]
};

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFFu) >> 4);          // start address, bits [0, 14)
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;       // leading (K-group) byte offset, [16, 30)
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;       // stride (MN-group) byte offset, [32, 46)
  d |= (uint64_t)1 << 46;                            // descriptor version 1 (sm_100)
  return d;                                          // base offset 0, no swizzle (layout 0)
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                                   // D format f32
         | (1u << 7) | (1u << 10)                    // A, B format bf16
         | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16)
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   nat::smem_u32(bar))
               : "memory");
}

// 16-byte asynchronous global -> shared copy (cp.async, LDGSTS); zero-filled outside the
// matrix (src-size 0)
__device__ __forceinline__ void cp16(char* dst, const bf16* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(nat::smem_u32(dst)),
               "l"(ok ? src : nullptr), "r"(ok ? 16 : 0)
               : "memory");
}

// Stages rows [r0, r0 + R) x k [k0, k0 + 64) of an operand into the core-matrix layout:
//   K-major : unit (r, kc) at ((r/8)*8 + kc)*128 + (r%8)*16   (LBO = 128, SBO = 1024)
//   MN-major: unit (kk, rc) at ((kk/8)*(R/8) + rc)*128 + (kk%8)*16 (SBO = 128, LBO = R*16)
template <int R, bool MN>
__device__ __forceinline__ void stage_operand(const bf16* P, int64_t ld, int64_t rows, int64_t K, int64_t r0,
                                              int64_t k0, char* smem) {
  constexpr int kUnits = R * (kBK / 8);
#pragma unroll 4
  for (int u = threadIdx.x; u < kUnits; u += kGT) {
    if constexpr (!MN) {
      const int r = u / (kBK / 8), kc = u % (kBK / 8);
      const int64_t gr = r0 + r, gk = k0 + kc * 8;
      cp16(smem + ((r / 8) * (kBK / 8) + kc) * 128 + (r % 8) * 16, P + gr * ld + gk, gr < rows && gk < K);
    } else {
      const int kk = u / (R / 8), rc = u % (R / 8);
      const int64_t gk = k0 + kk, gr = r0 + rc * 8;
      cp16(smem + ((kk / 8) * (R / 8) + rc) * 128 + (kk % 8) * 16, P + gk * ld + gr, gk < K && gr < rows);
    }
  }
}

// cp.async.wait_group with a run-time count (immediate operand): groups still allowed in flight
__device__ __forceinline__ void cp_wait_pending(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

// shared-memory stages of the operand pipeline (<= 4; 3 for the 128-wide tiles so that two
// CTAs share an SM)
template <int BN>
constexpr int gemm_stages() {
  return BN >= 128 ? 3 : 4;
}

// Epilogue of one 128 x BN tile from TMEM (accumulator at column `tmem`): warp w owns rows
// (TMEM lanes) 32 (w % 4) .. + 31 and column half w / 4 (BN >= 64; narrower tiles: warps 0-3
// take all columns); 32 columns per tcgen05.ld.  colsum[4][BN] receives the masked
// gradient's column sums per lane quarter (kEpiMaskBf16).
template <int BN>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& g, uint32_t tmem, int64_t m0, int split, bool have,
                                              const float* bias_s, float (*colsum)[BN]) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wq = warp & 3, ch = warp >> 2;
  const int64_t m = m0 + wq * 32 + lane;
  const bool row_ok = m < g.M && have;
  constexpr int kHalf = BN >= 64 ? BN / 2 : BN;
  const bool epi_warp = BN >= 64 || ch == 0;
#pragma unroll 1
  for (int n0 = ch * kHalf; epi_warp && n0 < (ch + 1) * kHalf; n0 += 32) {
    constexpr int WH = BN < 32 ? BN : 32;
    uint4 hv[WH / 8];  // the ReLU mask's row slice, loaded ahead of the TMEM read (latency overlap)
    if (g.epi == kEpiMaskBf16) {
#pragma unroll
      for (int q = 0; q < WH / 8; ++q)
        hv[q] = row_ok ? *reinterpret_cast<const uint4*>(g.H + m * g.ldh + n0 + 8 * q) : make_uint4(0, 0, 0, 0);
    }
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)n0;
    if constexpr (BN >= 32) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
            "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
            "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
    } else {  // BN == 16
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
            "=r"(v[15])
          : "r"(taddr));
      for (int q = 16; q < 32; ++q) v[q] = 0u;
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    constexpr int W = BN < 32 ? BN : 32;
    float f[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) f[q] = __uint_as_float(v[q]);
    if (g.epi == kEpiBiasReluBf16 || g.epi == kEpiMaskBf16) {
      if (g.epi == kEpiBiasReluBf16) {
#pragma unroll
        for (int q = 0; q < W; ++q) f[q] = fmaxf(f[q] + bias_s[n0 + q], 0.f);
      } else {
#pragma unroll
        for (int q = 0; q < W; q += 8) {
          const bf16* hb = reinterpret_cast<const bf16*>(&hv[q / 8]);
#pragma unroll
          for (int e = 0; e < 8; ++e) f[q + e] = (row_ok && __bfloat162float(hb[e]) > 0.f) ? f[q + e] : 0.f;
        }
        // column sums of the masked gradient (bias gradient): a transposing butterfly over the
        // warp (31 shuffles for 32 columns; lane l ends with column l's sum over the 32 rows),
        // then the 4 lane quarters in order
        if constexpr (W == 32) {
          float t[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) t[q] = f[q];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int q = 0; q < o; ++q) {
              const float send = up ? t[q] : t[q + o];
              const float recv = __shfl_xor_sync(0xffffffffu, send, o);
              t[q] = (up ? t[q + o] : t[q]) + recv;
            }
          }
          colsum[wq][n0 + lane] = t[0];
        } else {
#pragma unroll
          for (int q = 0; q < W; ++q) {
            float t = f[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) colsum[wq][n0 + q] = t;
          }
        }
      }
      if (row_ok) {
#pragma unroll
        for (int q = 0; q < W; q += 8) {
          uint4 o;
          __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
          for (int e = 0; e < 4; ++e) ob[e] = __floats2bfloat162_rn(f[q + 2 * e], f[q + 2 * e + 1]);
          *reinterpret_cast<uint4*>(g.Cb + m * g.ldc + n0 + q) = o;
        }
      }
    } else if (g.epi == kEpiPartial) {
      if (row_ok) {
        float* dst = g.C + ((size_t)split * g.M + m) * g.ldc + n0;
#pragma unroll
        for (int q = 0; q < W; q += 4) *reinterpret_cast<float4*>(dst + q) = make_float4(f[q], f[q + 1], f[q + 2], f[q + 3]);
      }
    } else {  // kEpiBiasF32, kEpiF32
      if (g.epi == kEpiBiasF32) {
#pragma unroll
        for (int q = 0; q < W; ++q) f[q] += bias_s[n0 + q];
      }
      if (row_ok) {
        float* dst = g.C + m * g.ldc + n0;
        if (n0 + W <= g.n_valid && (g.ldc % 4) == 0) {
#pragma unroll
          for (int q = 0; q < W; q += 4) *reinterpret_cast<float4*>(dst + q) = make_float4(f[q], f[q + 1], f[q + 2], f[q + 3]);
        } else {
          for (int q = 0; q < W; ++q)
            if (n0 + q < g.n_valid) dst[q] = f[q];
        }
      }
    }
  }
}

template <int BN, bool AMN, bool BMN>
__global__ void __launch_bounds__(kGT) nf_gemm_kernel(GemmArgs g) {
  constexpr uint32_t kABytes = kGM * kBK * 2, kBBytes = BN * kBK * 2;
  constexpr uint32_t kCols = BN < 32 ? 32 : BN;  // TMEM columns (power of 2 >= 32)
  constexpr int S = gemm_stages<BN>();
  extern __shared__ __align__(1024) char gsm[];
  __shared__ __align__(8) uint64_t bars[S];
  __shared__ uint32_t tmem_base;
  __shared__ float colsum[4][BN];
  __shared__ float bias_s[BN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wq = warp & 3, ch = warp >> 2;  // TMEM lane quarter, column half of the epilogue
  const int64_t m0 = (int64_t)blockIdx.x * kGM;
  const int split = blockIdx.y;
  const int64_t kb = (int64_t)split * g.k_per_cta, ke = min(g.K, kb + g.k_per_cta);
  const int nchunk = (int)((ke - kb + kBK - 1) / kBK);
  auto sA = [&](int st) { return gsm + (size_t)st * (kABytes + kBBytes); };
  auto sB = [&](int st) { return gsm + (size_t)st * (kABytes + kBBytes) + kABytes; };
  // chunk c -> stage c % S: both operands' 16-byte pieces, one cp.async group per chunk
  auto stage = [&](int c) {
    const int64_t k0 = kb + (int64_t)c * kBK;
    stage_operand<kGM, AMN>(g.A, g.lda, g.M, ke, m0, k0, sA(c % S));
    stage_operand<BN, BMN>(g.B, g.ldb, g.N, ke, 0, k0, sB(c % S));
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if (tid == 0) {
    for (int q = 0; q < S; ++q) nat::mbar_init(&bars[q], 1);
    nat::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(nat::smem_u32(&tmem_base)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // the first S chunks' loads are in flight before the TMEM handshake completes
  for (int c = 0; c < S && c < nchunk; ++c) stage(c);
  if (g.bias)
    for (int n = tid; n < BN; n += kGT) bias_s[n] = n < g.n_bias ? g.bias[n] : 0.f;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = idesc_bf16(kGM, BN, AMN, BMN);
  // descriptor strides (bytes): K-group (LBO) and MN-group (SBO)
  constexpr uint32_t a_lbo = AMN ? kGM * 16 : 128, a_sbo = AMN ? 128 : (kBK / 8) * 128;
  constexpr uint32_t b_lbo = BMN ? BN * 16 : 128, b_sbo = BMN ? 128 : (kBK / 8) * 128;

  for (int c = 0; c < nchunk; ++c) {
    // groups committed so far: min(nchunk, c + S); chunk c's is done when at most
    // min(nchunk, c + S) - (c + 1) younger ones are pending
    cp_wait_pending(min(nchunk, c + S) - (c + 1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> tensor core reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = nat::smem_u32(sA(c % S)), b0 = nat::smem_u32(sB(c % S));
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk)
        mma_bf16(tmem, sdesc(a0 + kk * 2 * a_lbo, a_lbo, a_sbo), sdesc(b0 + kk * 2 * b_lbo, b_lbo, b_sbo), idesc,
                 (c > 0 || kk > 0) ? 1u : 0u);
      mma_commit(&bars[c % S]);
    }
    if (c + S < nchunk) {  // refill this stage once its MMAs have read it
      nat::mbar_wait(&bars[c % S], (uint32_t)((c / S) & 1));
      stage(c + S);
    }
  }
  if (nchunk > 0) nat::mbar_wait(&bars[(nchunk - 1) % S], (uint32_t)(((nchunk - 1) / S) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;");

  gemm_epilogue<BN>(g, tmem, m0, split, nchunk > 0, bias_s, colsum);
  if (g.epi == kEpiMaskBf16) {
    __syncthreads();
    for (int n = tid; n < BN; n += kGT)
      g.colpart[(size_t)blockIdx.x * BN + n] = ((colsum[0][n] + colsum[1][n]) + colsum[2][n]) + colsum[3][n];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// Persistent variant for the products with K <= 128 over the batch (forward Y = X W^T and
// input gradients dX = dY W): A = activations [M][K] K-major, B = the layer's weights,
// staged ONCE per CTA.  The CTA walks the 128-row tiles t = blockIdx.x, + gridDim.x, ...
// with two A buffers and two TMEM accumulators: while tile i's MMAs run, tile i+1's rows
// are loading and tile i-1's epilogue drains its accumulator.
template <int BN, bool BMN>
__global__ void __launch_bounds__(kGT) nf_gemm_persist_kernel(GemmArgs g, int64_t n_tiles) {
  constexpr uint32_t kABytes = kGM * kBK * 2, kBBytes = BN * kBK * 2;
  constexpr uint32_t kCols = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) char gsm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  __shared__ float colsum[4][BN];
  __shared__ float bias_s[BN];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nchunk = (int)((g.K + kBK - 1) / kBK);  // 1 or 2
  char* sB = gsm;                                      // [2 chunks] weights
  auto sA = [&](int buf) { return gsm + 2 * kBBytes + (size_t)buf * 2 * kABytes; };
  const int64_t my_n = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto stage_a = [&](int64_t i) {
    const int64_t m0 = (blockIdx.x + i * gridDim.x) * (int64_t)kGM;
    for (int c = 0; c < nchunk; ++c)
      stage_operand<kGM, false>(g.A, g.lda, g.M, g.K, m0, (int64_t)c * kBK, sA((int)(i & 1)) + (size_t)c * kABytes);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (tid == 0) {
    nat::mbar_init(&bars[0], 1);
    nat::mbar_init(&bars[1], 1);
    nat::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(nat::smem_u32(&tmem_base)),
                 "r"(2 * kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (my_n > 0) {
    for (int c = 0; c < nchunk; ++c)
      stage_operand<BN, BMN>(g.B, g.ldb, g.N, g.K, 0, (int64_t)c * kBK, sB + (size_t)c * kBBytes);
    stage_a(0);  // group 0: weights + tile 0
    if (my_n > 1) stage_a(1);
  }
  if (g.bias)
    for (int n = tid; n < BN; n += kGT) bias_s[n] = n < g.n_bias ? g.bias[n] : 0.f;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem0 = tmem_base;
  constexpr uint32_t idesc = idesc_bf16(kGM, BN, false, BMN);
  constexpr uint32_t a_lbo = 128, a_sbo = (kBK / 8) * 128;
  constexpr uint32_t b_lbo = BMN ? BN * 16 : 128, b_sbo = BMN ? 128 : (kBK / 8) * 128;
  auto drain = [&](int64_t i) {  // epilogue of tile i (its MMAs are complete)
    const int64_t tile = blockIdx.x + i * gridDim.x;
    gemm_epilogue<BN>(g, tmem0 + (uint32_t)(i & 1) * kCols, tile * kGM, 0, true, bias_s, colsum);
    if (g.epi == kEpiMaskBf16) {
      __syncthreads();
      for (int n = tid; n < BN; n += kGT)
        g.colpart[(size_t)tile * BN + n] = ((colsum[0][n] + colsum[1][n]) + colsum[2][n]) + colsum[3][n];
    }
  };
  for (int64_t i = 0; i < my_n; ++i) {
    if (i == 0 && my_n > 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = nat::smem_u32(sA((int)(i & 1))), b0 = nat::smem_u32(sB);
      const uint32_t acc = tmem0 + (uint32_t)(i & 1) * kCols;
      for (int c = 0; c < nchunk; ++c)
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          mma_bf16(acc, sdesc(a0 + c * kABytes + kk * 2 * a_lbo, a_lbo, a_sbo),
                   sdesc(b0 + c * kBBytes + kk * 2 * b_lbo, b_lbo, b_sbo), idesc, (c > 0 || kk > 0) ? 1u : 0u);
      mma_commit(&bars[i & 1]);
    }
    if (i >= 1) {
      nat::mbar_wait(&bars[(i - 1) & 1], (uint32_t)(((i - 1) >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (i + 1 < my_n) stage_a(i + 1);  // into the buffer tile i-1's MMAs have released
      drain(i - 1);
    }
  }
  if (my_n > 0) {
    nat::mbar_wait(&bars[(my_n - 1) & 1], (uint32_t)(((my_n - 1) >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;");
    drain(my_n - 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem0), "r"(2 * kCols));
}

template <int BN, bool BMN>
cudaError_t launch_persist_t(const GemmArgs& g, cudaStream_t s) {
  const size_t smem = 2 * ((size_t)BN * kBK * 2) + 2 * 2 * ((size_t)kGM * kBK * 2);
  auto k = nf_gemm_persist_kernel<BN, BMN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (g.M + kGM - 1) / kGM;
  const int64_t grid = std::min<int64_t>(tiles, 2 * (int64_t)nat::device_sm_count());
  k<<<(unsigned)grid, kGT, smem, s>>>(g, tiles);
  return cudaGetLastError();
}

template <int BN, bool AMN, bool BMN>
cudaError_t launch_gemm_t(const GemmArgs& g, int splits, cudaStream_t s) {
  const size_t smem = (size_t)gemm_stages<BN>() * ((size_t)kGM * kBK * 2 + (size_t)BN * kBK * 2);
  auto k = nf_gemm_kernel<BN, AMN, BMN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((g.M + kGM - 1) / kGM), (unsigned)splits);
  k<<<grid, kGT, smem, s>>>(g);
  return cudaGetLastError();
}

template <bool AMN, bool BMN>
cudaError_t launch_gemm_n(const GemmArgs& g, int splits, cudaStream_t s) {
  switch (g.N) {
    case 16: return launch_gemm_t<16, AMN, BMN>(g, splits, s);
    case 32: return launch_gemm_t<32, AMN, BMN>(g, splits, s);
    case 64: return launch_gemm_t<64, AMN, BMN>(g, splits, s);
    case 128: return launch_gemm_t<128, AMN, BMN>(g, splits, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm(const GemmArgs& g, bool a_mn, bool b_mn, int splits, cudaStream_t s) {
  const bool timed = nat::ktimer_on();  // diagnostics: flops = 2 M N K of the product
  if (timed) nat::ktimer_begin(nat::kTimerNfGemm, s);
  cudaError_t e;
  static const bool persist_env = [] {  // NAT_NF_PERSIST=0: the one-tile-per-CTA kernel (A/B)
    const char* v = std::getenv("NAT_NF_PERSIST");
    return !(v && v[0] == '0');
  }();
  if (persist_env && !a_mn && splits == 1 && g.K <= 2 * kBK && g.k_per_cta >= g.K) {
    switch (g.N) {
      case 16: e = b_mn ? launch_persist_t<16, true>(g, s) : launch_persist_t<16, false>(g, s); break;
      case 32: e = b_mn ? launch_persist_t<32, true>(g, s) : launch_persist_t<32, false>(g, s); break;
      case 64: e = b_mn ? launch_persist_t<64, true>(g, s) : launch_persist_t<64, false>(g, s); break;
      case 128: e = b_mn ? launch_persist_t<128, true>(g, s) : launch_persist_t<128, false>(g, s); break;
      default: e = cudaErrorInvalidValue;
    }
  } else if (!a_mn && !b_mn) e = launch_gemm_n<false, false>(g, splits, s);
  else if (!a_mn && b_mn) e = launch_gemm_n<false, true>(g, splits, s);
  else if (a_mn && !b_mn) e = launch_gemm_n<true, false>(g, splits, s);
  else e = launch_gemm_n<true, true>(g, splits, s);
  if (timed) nat::ktimer_end(nat::kTimerNfGemm, s, 2.0 * (double)g.M * (double)g.N * (double)g.K, nullptr);
  return e;
}

// =====================================================================================
// encoding, loss, grid scatter, reductions, Adam
// =====================================================================================
// X[b][0..16) = grid features (level-major), X[b][16..16 + 12 n_v) = PE(v), rest 0 (bf16)
__global__ void nf_encode_kernel(int64_t n, int n_v, const float* __restrict__ in, const float* __restrict__ params,
                                 Layout L, bf16* __restrict__ X) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  const float* x = in + b * (3 + n_v);
  float out[kInPad];
#pragma unroll
  for (int q = 0; q < kInPad; ++q) out[q] = 0.f;
#pragma unroll
  for (int l = 0; l < kLevels; ++l) {
    const int N = level_res(l);
    int64_t i0[3];
    float fr[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float p = x[d] * (float)N;
      const float fl = fminf(fmaxf(floorf(p), 0.f), (float)(N - 1));
      i0[d] = (int64_t)fl;
      fr[d] = p - fl;
    }
    const float* G = params + L.grid[l];
    float acc[kFeat] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
      const float wx = dx ? fr[0] : 1.f - fr[0], wy = dy ? fr[1] : 1.f - fr[1], wz = dz ? fr[2] : 1.f - fr[2];
      const float w = __fmul_rn(__fmul_rn(wx, wy), wz);
      const float4 f = *reinterpret_cast<const float4*>(G + vertex_row(l, i0[0] + dx, i0[1] + dy, i0[2] + dz) * kFeat);
      acc[0] = __fadd_rn(acc[0], __fmul_rn(w, f.x));
      acc[1] = __fadd_rn(acc[1], __fmul_rn(w, f.y));
      acc[2] = __fadd_rn(acc[2], __fmul_rn(w, f.z));
      acc[3] = __fadd_rn(acc[3], __fmul_rn(w, f.w));
    }
#pragma unroll
    for (int f = 0; f < kFeat; ++f) out[l * kFeat + f] = acc[f];
  }
  for (int d = 0; d < n_v; ++d)
    for (int k = 0; k < kPeFreq; ++k) {
      const float a = (float)(1 << k) * 3.14159265358979323846f * x[3 + d];
      float sn, cs;
      sincosf(a, &sn, &cs);
      out[kLevels * kFeat + 2 * (d * kPeFreq + k)] = sn;
      out[kLevels * kFeat + 2 * (d * kPeFreq + k) + 1] = cs;
    }
  uint4* dst = reinterpret_cast<uint4*>(X + b * kInPad);
#pragma unroll
  for (int q = 0; q < kInPad; q += 8) {
    uint4 o;
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) ob[e] = __floats2bfloat162_rn(out[q + 2 * e], out[q + 2 * e + 1]);
    dst[q / 8] = o;
  }
}

// dY = 2 (Y - T) / (n n_out) (bf16 [n][16], zero padded); per-block partial sums of the
// squared error (loss) and of dY per column (output-layer bias gradient), fixed order.
constexpr int kLossT = 256;
__global__ void __launch_bounds__(kLossT) nf_loss_kernel(int64_t n, int n_out, const float* __restrict__ Y,
                                                         const float* __restrict__ T, bf16* __restrict__ dY,
                                                         double* __restrict__ lpart, float* __restrict__ bpart) {
  __shared__ double sl[kLossT];
  __shared__ float sb[kOutPad][kLossT / 32];
  const int64_t b = blockIdx.x * (int64_t)kLossT + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double se = 0.0;
  float d[kOutPad];
#pragma unroll
  for (int q = 0; q < kOutPad; ++q) d[q] = 0.f;
  if (b < n) {
    const float scale = 2.f / (float)((double)n * n_out);
    for (int q = 0; q < n_out; ++q) {
      const float e = Y[b * kOutPad + q] - T[b * n_out + q];
      se += (double)e * (double)e;
      d[q] = scale * e;
    }
    uint4 o[2];
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(o);
#pragma unroll
    for (int e = 0; e < 8; ++e) ob[e] = __floats2bfloat162_rn(d[2 * e], d[2 * e + 1]);
    reinterpret_cast<uint4*>(dY + b * kOutPad)[0] = o[0];
    reinterpret_cast<uint4*>(dY + b * kOutPad)[1] = o[1];
  }
  sl[threadIdx.x] = se;
#pragma unroll
  for (int q = 0; q < kOutPad; ++q) {
    float t = d[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) sb[q][warp] = t;
  }
  __syncthreads();
  for (int w = kLossT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sl[threadIdx.x] += sl[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) lpart[blockIdx.x] = sl[0];
  if (threadIdx.x < kOutPad) {
    float t = 0.f;
    for (int w = 0; w < kLossT / 32; ++w) t += sb[threadIdx.x][w];
    bpart[(size_t)blockIdx.x * kOutPad + threadIdx.x] = t;
  }
}

// Split-K / per-tile partial sums: out[j] = sum_p part[p][j] in a fixed order.
// transpose: out holds [cols][rows] of a [rows][cols] partial layout (dW of the last layer).
// 8 partial groups per output (group g takes p = g, g + 8, ... in
// ascending order, then the 8 group sums in group order): deterministic, coalesced over
// 32 consecutive outputs per block.
__global__ void __launch_bounds__(256) nf_reduce_wide_kernel(int64_t nparts, int64_t rows, int64_t cols,
                                                             const float* __restrict__ part, float* __restrict__ out,
                                                             int64_t out_rows, int64_t out_cols, bool transpose) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32 + lane;
  const int64_t total = rows * cols;
  float t = 0.f;
  if (j < total) {
    int64_t p = grp;
    for (; p + 24 < nparts; p += 32) {
      const float a = part[p * total + j], b = part[(p + 8) * total + j], c = part[(p + 16) * total + j],
                  d = part[(p + 24) * total + j];
      t = (((t + a) + b) + c) + d;
    }
    for (; p < nparts; p += 8) t += part[p * total + j];
  }
  sm[grp][lane] = t;
  __syncthreads();
  if (grp == 0 && j < total) {
    float u = sm[0][lane];
    for (int g = 1; g < 8; ++g) u += sm[g][lane];
    const int64_t r = j / cols, c = j % cols;
    if (!transpose) {
      if (r < out_rows && c < out_cols) out[r * out_cols + c] = u;
    } else {
      if (c < out_rows && r < out_cols) out[c * out_cols + r] = u;
    }
  }
}

// First level of a tall reduction (many parts, few columns): block (x, y) sums the parts
// [y per, (y + 1) per) of columns x*32 .. x*32 + 31 (8 groups strided over the parts, then
// the groups in order) into tmp[y][j]; nf_reduce_wide_kernel then sums the gridDim.y rows.
__global__ void __launch_bounds__(256) nf_reduce_tall_kernel(int64_t nparts, int64_t total, int64_t per,
                                                             const float* __restrict__ part, float* __restrict__ tmp) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32 + lane;
  const int64_t p0 = blockIdx.y * per, p1 = min(nparts, p0 + per);
  float t = 0.f;
  if (j < total)
    for (int64_t p = p0 + grp; p < p1; p += 8) t += part[p * total + j];
  sm[grp][lane] = t;
  __syncthreads();
  if (grp == 0 && j < total) {
    float u = sm[0][lane];
    for (int g = 1; g < 8; ++g) u += sm[g][lane];
    tmp[blockIdx.y * total + j] = u;
  }
}

// one block: thread t sums parts t, t + 256, ... in order, then a fixed tree
__global__ void __launch_bounds__(256) nf_loss_finish_kernel(int64_t nparts, const double* __restrict__ lpart,
                                                             int64_t count, float* __restrict__ loss) {
  __shared__ double sm[256];
  double t = 0.0;
  for (int64_t p = threadIdx.x; p < nparts; p += 256) t += lpart[p];
  sm[threadIdx.x] = t;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = (float)(sm[0] / (double)count);
}

// dGrid[level][row] += w_corner * dX[b][level*4 + f]   (atomics: order-free sums).
// Persistent CTAs; the two coarse lattices (729 + 4913 rows, every sample hits them) are
// accumulated in shared memory and flushed once per CTA, the fine ones atomically in HBM.
constexpr int kSmemLevels = 2;
__host__ __device__ constexpr int64_t smem_grid_rows() { return level_rows(0) + level_rows(1); }

__global__ void __launch_bounds__(256) nf_grid_backward_kernel(int64_t n, int n_v, const float* __restrict__ in,
                                                               const float* __restrict__ dX, Layout L,
                                                               float* __restrict__ grad, int smem_levels) {
  extern __shared__ float sg[];  // [smem_grid_rows][4]
  for (int64_t i = threadIdx.x; i < smem_grid_rows() * kFeat; i += blockDim.x) sg[i] = 0.f;
  __syncthreads();
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const float* x = in + b * (3 + n_v);
#pragma unroll
    for (int l = 0; l < kLevels; ++l) {
      const int N = level_res(l);
      int64_t i0[3];
      float fr[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const float p = x[d] * (float)N;
        const float fl = fminf(fmaxf(floorf(p), 0.f), (float)(N - 1));
        i0[d] = (int64_t)fl;
        fr[d] = p - fl;
      }
      const float4 g = *reinterpret_cast<const float4*>(dX + b * kInPad + l * kFeat);
      const bool in_smem = l < smem_levels;
      float* G = in_smem ? sg + (l == 0 ? 0 : level_rows(0) * kFeat) : grad + L.grid[l];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int dx = c & 1, dy = (c >> 1) & 1, dz = (c >> 2) & 1;
        const float wx = dx ? fr[0] : 1.f - fr[0], wy = dy ? fr[1] : 1.f - fr[1], wz = dz ? fr[2] : 1.f - fr[2];
        const float w = (wx * wy) * wz;
        float* r = G + vertex_row(l, i0[0] + dx, i0[1] + dy, i0[2] + dz) * kFeat;
        if (in_smem) {
          atomicAdd(r + 0, w * g.x);
          atomicAdd(r + 1, w * g.y);
          atomicAdd(r + 2, w * g.z);
          atomicAdd(r + 3, w * g.w);
        } else {  // one 16-byte vector reduction (red.global.add.v4.f32) per corner
          atomicAdd(reinterpret_cast<float4*>(r), make_float4(w * g.x, w * g.y, w * g.z, w * g.w));
        }
      }
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < smem_grid_rows() * kFeat; i += blockDim.x) {
    const float v = sg[i];
    if (v != 0.f) {
      const int64_t l0 = level_rows(0) * kFeat;
      atomicAdd(grad + (i < l0 ? L.grid[0] + i : L.grid[1] + (i - l0)), v);
    }
  }
}

// Adam (Kingma & Ba) with bias correction; step counts from 1.
__global__ void nf_adam_kernel(int64_t n, float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                               float* __restrict__ v, float lr, float b1, float b2, float eps, float c1, float c2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = b1 * m[i] + (1.f - b1) * gi;
  const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
}

// bf16 copies of the layer weights: Wb_q [out_pad][in] (rows >= out zero)
__global__ void nf_cast_weights_kernel(const float* __restrict__ params, Layout L, bf16* __restrict__ Wb) {
  const int q = blockIdx.y;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int out_pad = q == kNHidden ? kOutPad : kHidden;
  const int64_t off = (int64_t)q * kHidden * kHidden;  // slot per layer
  if (j >= (int64_t)out_pad * L.in[q]) return;
  const int64_t r = j / L.in[q], c = j % L.in[q];
  Wb[off + j] = r < L.out[q] ? __float2bfloat16_rn(params[L.W[q] + r * L.in[q] + c]) : __float2bfloat16_rn(0.f);
}

struct NfWs {
  bf16* X;        // [n][64]
  bf16* H[kNHidden];  // [n][128]
  float* Y;       // [n][16]
  bf16* dY;       // [n][16]
  bf16* dH[2];    // [n][128]
  float* dX;      // [n][64]
  float* grad;    // [n_params]
  bf16* Wb;       // [5][128][128] bf16 weight slots
  float* wpart;   // [splits][128][128]
  float* cpart;   // [tiles][128]
  float* rtmp;    // [kTallRows][128] first level of the tall column-sum reductions
  double* lpart;  // loss partials
  float* bpart;   // [loss blocks][16]
  int64_t splits, tiles, lblocks;
};

// batch rows per split-K CTA of the weight gradients (NAT_NF_SPLIT_ROWS for A/B; default 1024)
int64_t split_rows() {
  static const int64_t v = [] {
    const char* e = std::getenv("NAT_NF_SPLIT_ROWS");
    const int64_t r = e ? std::atoll(e) : 1024;
    return r >= 128 && r % 64 == 0 ? r : (int64_t)1024;
  }();
  return v;
}
constexpr int kTallRows = 64;         // first-level rows of the tall column-sum reductions

// column sums of part[nparts][cols] (cols <= 128) -> out (fixed order, two levels)
void reduce_tall(int64_t nparts, int64_t cols, const float* part, float* out, int64_t out_cols, float* tmp,
                 cudaStream_t s) {
  const int64_t G = std::min<int64_t>(kTallRows, (nparts + 31) / 32);
  const int64_t per = (nparts + G - 1) / G;
  nf_reduce_tall_kernel<<<dim3((unsigned)((cols + 31) / 32), (unsigned)G), 256, 0, s>>>(nparts, cols, per, part, tmp);
  nf_reduce_wide_kernel<<<(unsigned)((cols + 31) / 32), 256, 0, s>>>(G, 1, cols, tmp, out, 1, out_cols, false);
}

size_t nf_carve(nat::Carver& c, NfWs* w, int64_t n, int64_t n_params) {
  NfWs t{};
  t.X = c.take<bf16>((size_t)n * kInPad);
  for (int q = 0; q < kNHidden; ++q) t.H[q] = c.take<bf16>((size_t)n * kHidden);
  t.Y = c.take<float>((size_t)n * kOutPad);
  t.dY = c.take<bf16>((size_t)n * kOutPad);
  t.dH[0] = c.take<bf16>((size_t)n * kHidden);
  t.dH[1] = c.take<bf16>((size_t)n * kHidden);
  t.dX = c.take<float>((size_t)n * kInPad);
  t.grad = c.take<float>((size_t)n_params);
  t.Wb = c.take<bf16>((size_t)kNLayers * kHidden * kHidden);
  t.splits = (n + split_rows() - 1) / split_rows();
  t.tiles = (n + kGM - 1) / kGM;
  t.lblocks = (n + kLossT - 1) / kLossT;
  t.wpart = c.take<float>((size_t)t.splits * kHidden * kHidden);
  t.cpart = c.take<float>((size_t)t.tiles * kHidden);
  t.rtmp = c.take<float>((size_t)kTallRows * kHidden);
  t.lpart = c.take<double>((size_t)t.lblocks);
  t.bpart = c.take<float>((size_t)t.lblocks * kOutPad);
  if (w) *w = t;
  return c.bytes();
}

nat_status check_cfg(const nat_nf_config* cfg) {
  NAT_REQUIRE(cfg, "cfg must be non-null");
  NAT_REQUIRE(cfg->n_v >= 0 && 16 + 12 * cfg->n_v <= kInPad, "n_v = %d: need 16 + 12 n_v <= 64", cfg->n_v);
  NAT_REQUIRE(cfg->n_out >= 1 && cfg->n_out <= kOutPad, "n_out = %d must be in [1, 16]", cfg->n_out);
  return NAT_OK;
}

#define NF_LAUNCH(expr)                                                                        \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess) return nat::fail(NAT_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// =====================================================================================
// Fused forward: all five layer products of a 128-sample tile in one persistent CTA.  The
// five bf16 weight matrices stay in shared memory (core-matrix K-major layout, 116 KB); a
// tile's activations never leave the SM between layers: each epilogue (bias + ReLU + bf16)
// writes its output both to global memory (H_q, kept for the backward pass) and into the
// next layer's A operand in shared memory; the next tile's input rows load (cp.async) while
// the current tile runs its chain.  One TMEM accumulator of 128 columns.
// =====================================================================================
struct FwdArgs {
  const bf16* X;        // [n][64]
  const bf16* Wb;       // [5][128][128] slots: W_q [out_pad][in]
  const float* bias[kNLayers];
  int n_bias[kNLayers];
  bf16* H[kNHidden];    // [n][128]
  float* Y;             // [n][16]
  int n_out;
  int64_t n;
};
constexpr uint32_t kFwdW0 = 128 * 64 * 2, kFwdWh = 128 * 128 * 2, kFwdW4 = 16 * 128 * 2;
constexpr uint32_t kFwdX = kGM * 64 * 2, kFwdH = kGM * 128 * 2;
constexpr uint32_t kFwdSmem = kFwdW0 + 3 * kFwdWh + kFwdW4 + 2 * kFwdX + 2 * kFwdH;  // two warpgroups' buffers

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Two warpgroups, two tiles in flight: warpgroup g (warps 4g .. 4g + 3, one per TMEM lane
// quarter) runs the layer chain of every other tile of the CTA with its own TMEM
// accumulator (columns 128 g ..), its own input and activation buffers, its own mbarrier and
// named barrier, so one group's epilogue overlaps the other group's tensor-core products.
// A layer's epilogue overwrites the group's activation buffer in place: the product that
// read it has completed (mbarrier) before the epilogue starts.
__device__ __forceinline__ void wg_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(128) : "memory");
}

__global__ void __launch_bounds__(kGT, 1) nf_forward_fused_kernel(FwdArgs a, int64_t n_tiles) {
  extern __shared__ __align__(1024) char fsm[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_base;
  __shared__ float bias_s[kNLayers][kHidden];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = warp >> 2, wq = warp & 3, gt = tid & 127;  // warpgroup, TMEM lane quarter, thread in group
  char* sW0 = fsm;
  char* sWh = sW0 + kFwdW0;                 // W1..W3
  char* sW4 = sWh + 3 * kFwdWh;
  char* sX = sW4 + kFwdW4 + (size_t)wg * kFwdX;
  char* sH = sW4 + kFwdW4 + 2 * kFwdX + (size_t)wg * kFwdH;
  const int64_t my_n = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // this group's tiles: i = wg, wg + 2, ... of the CTA's
  auto tile_row0 = [&](int64_t i) { return (blockIdx.x + i * gridDim.x) * (int64_t)kGM; };
  auto stage_x = [&](int64_t i) {  // 128 threads of the group stage the tile's input rows
    const int64_t m0 = tile_row0(i);
    constexpr int kUnits = kGM * (kBK / 8);
#pragma unroll 4
    for (int u = gt; u < kUnits; u += 128) {
      const int r = u / (kBK / 8), kc = u % (kBK / 8);
      const int64_t gr = m0 + r;
      cp16(sX + ((r / 8) * (kBK / 8) + kc) * 128 + (r % 8) * 16, a.X + gr * kInPad + kc * 8, gr < a.n);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (tid == 0) {
    nat::mbar_init(&bars[0], 1);
    nat::mbar_init(&bars[1], 1);
    nat::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(nat::smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (my_n > 0) {  // weights, then each group's first tile
    stage_operand<128, false>(a.Wb, kInPad, 128, kInPad, 0, 0, sW0);
    for (int q = 1; q <= 3; ++q)
      for (int c = 0; c < 2; ++c)
        stage_operand<128, false>(a.Wb + (size_t)q * kHidden * kHidden, kHidden, 128, kHidden, 0, c * kBK,
                                  sWh + (size_t)(q - 1) * kFwdWh + c * (kFwdWh / 2));
    for (int c = 0; c < 2; ++c)
      stage_operand<16, false>(a.Wb + (size_t)kNHidden * kHidden * kHidden, kHidden, 16, kHidden, 0, c * kBK,
                               sW4 + c * (kFwdW4 / 2));
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (wg < my_n) stage_x(wg);
  }
  for (int q = 0; q < kNLayers; ++q)
    for (int c = tid; c < kHidden; c += kGT) bias_s[q][c] = c < a.n_bias[q] ? a.bias[q][c] : 0.f;
  asm volatile("cp.async.wait_all;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base + (uint32_t)wg * 128;
  uint64_t* bar = &bars[wg];
  uint32_t phase = 0;
  // one layer product of this group: acc = A [128 x K] * W^T (K-major core layout, chunks of 64)
  auto mma = [&](const char* A, uint32_t a_chunk, const char* W, uint32_t w_chunk, int nchunk, int N) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    wg_sync(wg);
    if (gt == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = nat::smem_u32(A), w0 = nat::smem_u32(W);
      const uint32_t idesc = N == 128 ? idesc_bf16(kGM, 128, false, false) : idesc_bf16(kGM, 16, false, false);
      for (int c = 0; c < nchunk; ++c)
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          mma_bf16(tmem, sdesc(a0 + c * a_chunk + kk * 256, 128, (kBK / 8) * 128),
                   sdesc(w0 + c * w_chunk + kk * 256, 128, (kBK / 8) * 128), idesc, (c > 0 || kk > 0) ? 1u : 0u);
      mma_commit(bar);
    }
    nat::mbar_wait(bar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
  };
  for (int64_t i = wg; i < my_n; i += 2) {
    const int64_t m = tile_row0(i) + wq * 32 + lane;
    const bool row_ok = m < a.n;
    asm volatile("cp.async.wait_all;" ::: "memory");  // this tile's input rows
    for (int q = 0; q < kNLayers; ++q) {
      if (q == 0) mma(sX, kFwdX, sW0, kFwdW0, 1, 128);
      else if (q < kNHidden) mma(sH, kFwdH / 2, sWh + (size_t)(q - 1) * kFwdWh, kFwdWh / 2, 2, 128);
      else mma(sH, kFwdH / 2, sW4, kFwdW4 / 2, 2, 16);
      if (q == 0 && i + 2 < my_n) stage_x(i + 2);  // the input buffer is free once product 0 is done
      if (q < kNHidden) {  // warp wq: rows 32 wq + lane, all 128 columns
#pragma unroll 1
        for (int n0 = 0; n0 < kHidden; n0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)n0, v);
          float f[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = fmaxf(__uint_as_float(v[e]) + bias_s[q][n0 + e], 0.f);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 o;
            __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) ob[e] = __floats2bfloat162_rn(f[8 * u + 2 * e], f[8 * u + 2 * e + 1]);
            if (row_ok) *reinterpret_cast<uint4*>(a.H[q] + m * kHidden + n0 + 8 * u) = o;
            // next product's A operand, in place: row r = 32 wq + lane, K unit (n0 + 8u) / 8
            const int r = wq * 32 + lane, kunit = (n0 + 8 * u) / 8;
            *reinterpret_cast<uint4*>(sH + (size_t)(kunit / 8) * (kFwdH / 2) + ((r / 8) * 8 + kunit % 8) * 128 +
                                      (r % 8) * 16) = row_ok ? o : make_uint4(0, 0, 0, 0);
          }
        }
      } else {  // output layer: 16 columns, fp32
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(wq * 32) << 16), v);
        if (row_ok) {
          float* y = a.Y + m * kOutPad;
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            *reinterpret_cast<float4*>(y + e) =
                make_float4(__uint_as_float(v[e]) + bias_s[q][e], __uint_as_float(v[e + 1]) + bias_s[q][e + 1],
                            __uint_as_float(v[e + 2]) + bias_s[q][e + 2], __uint_as_float(v[e + 3]) + bias_s[q][e + 3]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256));
}

cudaError_t launch_forward_fused(const FwdArgs& fa, cudaStream_t s) {
  auto k = nf_forward_fused_kernel;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwdSmem);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (fa.n + kGM - 1) / kGM;
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)nat::device_sm_count());
  const bool timed = nat::ktimer_on();
  if (timed) nat::ktimer_begin(nat::kTimerNfGemm, s);
  k<<<(unsigned)grid, kGT, kFwdSmem, s>>>(fa, tiles);
  e = cudaGetLastError();
  if (timed) {  // flops of the five products
    const double n = (double)fa.n;
    nat::ktimer_end(nat::kTimerNfGemm, s,
                    2.0 * n * (kHidden * (double)kInPad + 3.0 * kHidden * kHidden + (double)kOutPad * kHidden), nullptr);
  }
  return e;
}

// forward through the 5 layers (weights already cast); H[q] stored for the backward pass
nat_status forward_impl(const Layout& L, int64_t n, const float* params, NfWs& w, cudaStream_t s) {
  static const bool fused = [] {  // NAT_NF_FUSED=0: the five layer products as separate launches (A/B)
    const char* e = std::getenv("NAT_NF_FUSED");
    return !(e && e[0] == '0');
  }();
  if (fused) {
    FwdArgs fa{};
    fa.X = w.X;
    fa.Wb = w.Wb;
    for (int q = 0; q < kNLayers; ++q) {
      fa.bias[q] = params + L.b[q];
      fa.n_bias[q] = L.out[q];
    }
    for (int q = 0; q < kNHidden; ++q) fa.H[q] = w.H[q];
    fa.Y = w.Y;
    fa.n_out = L.out[kNHidden];
    fa.n = n;
    NF_LAUNCH(launch_forward_fused(fa, s));
    return NAT_OK;
  }
  const bf16* act = w.X;
  for (int q = 0; q < kNLayers; ++q) {
    GemmArgs g{};
    g.A = act;
    g.lda = L.in[q];
    g.B = w.Wb + (size_t)q * kHidden * kHidden;
    g.ldb = L.in[q];
    g.M = n;
    g.K = L.in[q];
    g.k_per_cta = L.in[q];
    g.bias = params + L.b[q];
    g.n_bias = L.out[q];
    if (q < kNHidden) {
      g.N = kHidden;
      g.epi = kEpiBiasReluBf16;
      g.Cb = w.H[q];
      g.ldc = kHidden;
      act = w.H[q];
    } else {
      g.N = kOutPad;
      g.epi = kEpiBiasF32;
      g.n_valid = L.out[q];
      g.C = w.Y;
      g.ldc = kOutPad;
    }
    NF_LAUNCH(launch_gemm(g, false, false, 1, s));
  }
  return NAT_OK;
}

}  // namespace

extern "C" int64_t nat_nf_param_count(const nat_nf_config* cfg) {
  if (check_cfg(cfg) != NAT_OK) return -1;
  return layout_of(cfg->n_out).total;
}

extern "C" size_t nat_nf_workspace(const nat_nf_config* cfg, int64_t n) {
  if (check_cfg(cfg) != NAT_OK || n < 1) return 0;
  nat::Carver c(nullptr);
  return nf_carve(c, nullptr, n, layout_of(cfg->n_out).total);
}

extern "C" nat_status nat_nf_forward(const nat_nf_config* cfg, const float* params, int64_t n, const float* inputs,
                                     float* out, void* ws, size_t ws_bytes, nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = check_cfg(cfg);
  if (st != NAT_OK) return st;
  NAT_REQUIRE(n >= 1, "need n >= 1 samples");
  NAT_REQUIRE_DEV(params);
  NAT_REQUIRE_DEV(inputs);
  NAT_REQUIRE_DEV(out);
  NAT_REQUIRE_DEV(ws);
  const Layout L = layout_of(cfg->n_out);
  nat::Carver c(ws);
  NfWs w;
  const size_t need = nf_carve(c, &w, n, L.total);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  nf_cast_weights_kernel<<<dim3((kHidden * kHidden + 255) / 256, kNLayers), 256, 0, s>>>(params, L, w.Wb);
  nf_encode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, cfg->n_v, inputs, params, L, w.X);
  NAT_LAUNCH_CHECK();
  st = forward_impl(L, n, params, w, s);
  if (st != NAT_OK) return st;
  NAT_CUDA_TRY(cudaMemcpy2DAsync(out, sizeof(float) * cfg->n_out, w.Y, sizeof(float) * kOutPad,
                                 sizeof(float) * cfg->n_out, n, cudaMemcpyDeviceToDevice, s));
  return NAT_OK;
}

extern "C" nat_status nat_nf_train_step(const nat_nf_config* cfg, float* params, float* adam_m, float* adam_v,
                                        int step, float lr, int64_t n, const float* inputs, const float* targets,
                                        float* loss, float* grad_out, void* ws, size_t ws_bytes,
                                        nat_stream_t stream) {
  NAT_TRACE();
  nat_status st = check_cfg(cfg);
  if (st != NAT_OK) return st;
  NAT_REQUIRE(n >= 1 && step >= 1, "need n >= 1 samples and step >= 1");
  NAT_REQUIRE(lr >= 0.f && lr < 1e30f, "bad learning rate");
  NAT_REQUIRE_DEV(params);
  NAT_REQUIRE_DEV(adam_m);
  NAT_REQUIRE_DEV(adam_v);
  NAT_REQUIRE_DEV(inputs);
  NAT_REQUIRE_DEV(targets);
  NAT_REQUIRE_DEV(loss);
  NAT_REQUIRE_DEV(ws);
  if (grad_out) NAT_REQUIRE_DEV(grad_out);
  const Layout L = layout_of(cfg->n_out);
  nat::Carver c(ws);
  NfWs w;
  const size_t need = nf_carve(c, &w, n, L.total);
  if (ws_bytes < need) return nat::fail(NAT_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  nf_cast_weights_kernel<<<dim3((kHidden * kHidden + 255) / 256, kNLayers), 256, 0, s>>>(params, L, w.Wb);
  nf_encode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, cfg->n_v, inputs, params, L, w.X);
  NAT_LAUNCH_CHECK();
  st = forward_impl(L, n, params, w, s);
  if (st != NAT_OK) return st;
  // loss and dY (MSE, l.124)
  nf_loss_kernel<<<(unsigned)w.lblocks, kLossT, 0, s>>>(n, cfg->n_out, w.Y, targets, w.dY, w.lpart, w.bpart);
  nf_loss_finish_kernel<<<1, 256, 0, s>>>(w.lblocks, w.lpart, n * cfg->n_out, loss);
  NAT_CUDA_TRY(cudaMemsetAsync(w.grad, 0, sizeof(float) * L.total, s));
  // output-layer bias gradient: column sums of dY
  reduce_tall(w.lblocks, kOutPad, w.bpart, w.grad + L.b[kNHidden], L.out[kNHidden], w.rtmp, s);
  // backward through the layers: d = gradient with respect to layer q's output
  const bf16* d = w.dY;
  int dcols = kOutPad;
  for (int q = kNHidden; q >= 0; --q) {
    const bf16* h_in = q == 0 ? w.X : w.H[q - 1];
    const int in = L.in[q];
    // dW_q = d^T h_in  (split-K over the batch): M = out (or in for the 16-wide last layer)
    GemmArgs gw{};
    gw.K = n;
    gw.k_per_cta = split_rows();
    gw.epi = kEpiPartial;
    gw.C = w.wpart;
    if (q == kNHidden) {  // C[in][out_pad] = h_in^T d: A = h_in (MN-major), B = dY (MN-major)
      gw.A = h_in;
      gw.lda = in;
      gw.M = in;
      gw.B = d;
      gw.ldb = dcols;
      gw.N = kOutPad;
      gw.ldc = kOutPad;
    } else {  // C[out][in] = d^T h_in
      gw.A = d;
      gw.lda = dcols;
      gw.M = kHidden;
      gw.B = h_in;
      gw.ldb = in;
      gw.N = in;
      gw.ldc = in;
    }
    NF_LAUNCH(launch_gemm(gw, true, true, (int)w.splits, s));
    const int64_t rows = gw.M, cols = gw.N;
    nf_reduce_wide_kernel<<<(unsigned)((rows * cols + 31) / 32), 256, 0, s>>>(
        w.splits, rows, cols, w.wpart, w.grad + L.W[q], L.out[q], in, q == kNHidden);
    NAT_LAUNCH_CHECK();
    // d_in = (d W_q) * relu'(h_in): M = n, N = in, K = out; B = W_q as [K = out][N = in] (MN-major)
    GemmArgs gd{};
    gd.A = d;
    gd.lda = dcols;
    gd.B = w.Wb + (size_t)q * kHidden * kHidden;
    gd.ldb = in;
    gd.M = n;
    gd.N = in;
    gd.K = q == kNHidden ? kOutPad : kHidden;
    gd.k_per_cta = gd.K;
    if (q > 0) {
      gd.epi = kEpiMaskBf16;
      gd.H = h_in;
      gd.ldh = in;
      gd.Cb = w.dH[q & 1];
      gd.ldc = in;
      gd.colpart = w.cpart;
      NF_LAUNCH(launch_gemm(gd, false, true, 1, s));
      // bias gradient of layer q - 1: column sums of the masked gradient, tile order
      reduce_tall(w.tiles, kHidden, w.cpart, w.grad + L.b[q - 1], kHidden, w.rtmp, s);
      NAT_LAUNCH_CHECK();
      d = w.dH[q & 1];
      dcols = in;
    } else {
      gd.epi = kEpiF32;
      gd.n_valid = in;
      gd.C = w.dX;
      gd.ldc = kInPad;
      NF_LAUNCH(launch_gemm(gd, false, true, 1, s));
    }
  }
  {
    const size_t gsm = sizeof(float) * smem_grid_rows() * kFeat;
    NAT_CUDA_TRY(cudaFuncSetAttribute(nf_grid_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
    const int64_t ctas = std::min<int64_t>(2 * (int64_t)nat::device_sm_count(), (n + 255) / 256);
    static const int smem_levels = [] {  // NAT_NF_SMEM_LEVELS: coarse levels accumulated in shared memory
      const char* v = std::getenv("NAT_NF_SMEM_LEVELS");
      return v ? std::max(0, std::min(kSmemLevels, std::atoi(v))) : 1;  // level 0 only (A/B: 1.071 vs 1.080 ms)
    }();
    nf_grid_backward_kernel<<<(unsigned)ctas, 256, gsm, s>>>(n, cfg->n_v, inputs, w.dX, L, w.grad, smem_levels);
  }
  NAT_LAUNCH_CHECK();
  if (grad_out) NAT_CUDA_TRY(cudaMemcpyAsync(grad_out, w.grad, sizeof(float) * L.total, cudaMemcpyDeviceToDevice, s));
  const float b1 = 0.9f, b2 = 0.999f;
  const float c1 = 1.f - std::pow(b1, (float)step), c2 = 1.f - std::pow(b2, (float)step);
  nf_adam_kernel<<<(unsigned)((L.total + 255) / 256), 256, 0, s>>>(L.total, params, w.grad, adam_m, adam_v, lr, b1,
                                                                  b2, 1e-8f, c1, c2);
  NAT_LAUNCH_CHECK();
  return NAT_OK;
}

// The tensor-core product of the layers on its own (tests / benchmarks): C (fp32 [M][N]) =
// A * B^T with A [M][K] (a_mn = 0) or [K][M] (a_mn = 1) and B [N][K] (b_mn = 0) or [K][N]
// (b_mn = 1), bf16, N in {16, 32, 64, 128}, K any, leading dimensions multiples of 8.
extern "C" nat_status nat_nf_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn,
                                       const void* B, int64_t ldb, int b_mn, float* C, int64_t ldc,
                                       nat_stream_t stream) {
  NAT_TRACE();
  NAT_REQUIRE(M >= 1 && K >= 1 && (N == 16 || N == 32 || N == 64 || N == 128), "bad shape");
  NAT_REQUIRE(lda % 8 == 0 && ldb % 8 == 0 && ldc >= N, "leading dimensions must be multiples of 8");
  NAT_REQUIRE_DEV(A);
  NAT_REQUIRE_DEV(B);
  NAT_REQUIRE_DEV(C);
  GemmArgs g{};
  g.A = (const bf16*)A;
  g.lda = lda;
  g.B = (const bf16*)B;
  g.ldb = ldb;
  g.M = M;
  g.N = N;
  g.K = K;
  g.k_per_cta = (K + kBK - 1) / kBK * kBK;
  g.epi = kEpiF32;
  g.n_valid = (int)N;
  g.C = C;
  g.ldc = ldc;
  NF_LAUNCH(launch_gemm(g, a_mn != 0, b_mn != 0, 1, (cudaStream_t)stream));
  return NAT_OK;
}
