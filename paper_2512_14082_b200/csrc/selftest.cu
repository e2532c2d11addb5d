// selftest.cu — single-tile tcgen05 checks of every operand path the hot
// kernels rely on (exported as us_selftest_umma, exercised by tests/test_gpu_selftest.py):
//   mode 0: A K-major (TMA), B K-major (TMA)            D = A * B^T   (proxy Q.K^T, attention S)
//   mode 1: A K-major (TMA), B MN-major (TMA)           D = A * B     (attention P.V with V row-major)
//   mode 2: A in TMEM (tcgen05.st), B K-major (TMA)     D = A * B^T   (TS path)
//   mode 3: A written by threads into swizzled smem, B MN-major: the attention P.V path.
//   mode 4: A MN-major (TMA of A^T stored [K][M]), B MN-major: the transposed attention
//           O^T = V^T P^T path (V rows [key][d] are the MN-major A of M = d).
// M = 128, K = 128 (two 64-element swizzle atoms), N in {64, 128}.
#include <cuda_runtime.h>

#include "host_util.hpp"
#include "ptx.cuh"

namespace us {
namespace {

constexpr int kM = 128, kK = 128;

template <int N>
__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const uint16_t* __restrict__ A_glob, int mode, int bf16, float* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 32 KB  [kc][128 rows][128 B]
  uint8_t* sB = smem + kM * kK * 2;   // 32 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  const bool b_mn = (mode == 1 || mode == 3 || mode == 4);
  // ---- operand staging
  if (threadIdx.x == 0) {
    uint32_t bytes = N * kK * 2;
    if (mode <= 1 || mode == 4) bytes += kM * kK * 2;
    mbar_arrive_expect_tx(&bar_tma, bytes);
    if (mode <= 1)
      for (int kc = 0; kc < 2; ++kc) tma_load_2d(sA + kc * kM * 128, &tmA, &bar_tma, kc * 64, 0);
    if (mode == 4)  // [mc][128 K rows][128 B]
      for (int mc = 0; mc < 2; ++mc) tma_load_2d(sA + mc * kK * 128, &tmA, &bar_tma, mc * 64, 0);
    if (!b_mn) {
      for (int kc = 0; kc < 2; ++kc) tma_load_2d(sB + kc * N * 128, &tmB, &bar_tma, kc * 64, 0);
    } else {
      for (int nc = 0; nc < N / 64; ++nc) tma_load_2d(sB + nc * kK * 128, &tmB, &bar_tma, nc * 64, 0);
    }
  }
  if (mode == 2) {
    // thread r holds row r of A; pack 2 x 16-bit per TMEM column.
    const int r = threadIdx.x;
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    for (int c0 = 0; c0 < kK / 2; c0 += 16) {
      uint32_t v[16];
      for (int t = 0; t < 16; ++t) {
        const uint32_t lo = A_glob[r * kK + 2 * (c0 + t)];
        const uint32_t hi = A_glob[r * kK + 2 * (c0 + t) + 1];
        v[t] = lo | (hi << 16);
      }
      tmem_st16(tmem + lane_base + 128 + c0, v);
    }
    tmem_st_wait();
  }
  if (mode == 3) {
    const int r = threadIdx.x;
    for (int kc = 0; kc < 2; ++kc)
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 val = *reinterpret_cast<const uint4*>(A_glob + r * kK + kc * 64 + ch * 8);
        *reinterpret_cast<uint4*>(sA + kc * kM * 128 + sw128_offset(r, ch)) = val;
      }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // ---- MMA issue
  if (warp == 0) {
    mbar_wait(&bar_tma, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = idesc_f16(kM, N, bf16 ? 1 : 0, mode == 4, b_mn);
      for (int k = 0; k < kK / 16; ++k) {
        const int kc = k / 4, ks = k % 4;
        uint64_t bdesc;
        if (!b_mn)
          bdesc = sdesc_sw128(smem_u32(sB + kc * N * 128 + ks * 32), 16, 1024);
        else
          bdesc = sdesc_sw128(smem_u32(sB + k * 16 * 128), kK * 128, 1024);
        if (mode == 2) {
          umma_f16_ts(tmem, tmem + 128 + k * 8, bdesc, idesc, k > 0);
        } else if (mode == 4) {
          const uint64_t adesc = sdesc_sw128(smem_u32(sA + k * 16 * 128), kK * 128, 1024);
          umma_f16_ss(tmem, adesc, bdesc, idesc, k > 0);
        } else {
          const uint64_t adesc = sdesc_sw128(smem_u32(sA + kc * kM * 128 + ks * 32), 16, 1024);
          umma_f16_ss(tmem, adesc, bdesc, idesc, k > 0);
        }
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int t = 0; t < 16; ++t) D[row * N + c0 + t] = __uint_as_float(v[t]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

}  // namespace
}  // namespace us

extern "C" us_status us_selftest_umma(int mode, int N, int bf16, const void* A, const void* B,
                                      float* D, void* stream) {
  using namespace us;
  if (mode < 0 || mode > 4 || (N != 64 && N != 128)) {
    set_error("us_selftest_umma: bad mode/N");
    return US_ERR_INVALID_ARGUMENT;
  }
  CUtensorMap tmA{}, tmB{};
  us_status s = mode == 4 ? make_tmap_2d_16b(&tmA, A, kK, kM, kK, 64, bf16)
                          : make_tmap_2d_16b(&tmA, A, kM, kK, kM, 64, bf16);
  if (s != US_OK) return s;
  const bool b_mn = (mode == 1 || mode == 3 || mode == 4);
  s = b_mn ? make_tmap_2d_16b(&tmB, B, kK, N, kK, 64, bf16)
           : make_tmap_2d_16b(&tmB, B, N, kK, N, 64, bf16);
  if (s != US_OK) return s;
  const size_t smem = 64 * 1024 + 1024;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (N == 64) {
    cudaFuncSetAttribute(selftest_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    selftest_kernel<64><<<1, 128, smem, st>>>(tmA, tmB, static_cast<const uint16_t*>(A), mode, bf16, D);
  } else {
    cudaFuncSetAttribute(selftest_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    selftest_kernel<128><<<1, 128, smem, st>>>(tmA, tmB, static_cast<const uint16_t*>(A), mode, bf16, D);
  }
  US_LAUNCH_CHECK("us_selftest_umma");
  return US_OK;
}

// ---------------------------------------------------------------- MMA issue-rate probe
// One CTA per SM issues `iters` groups of `per_group` back-to-back tcgen05.mma
// (M=128, K=16, bf16) with shape N and operand mode, then waits for completion.
// The host converts elapsed time into cycles per MMA. Operands are arbitrary
// smem/TMEM contents (only timing matters).
namespace us {
namespace {
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int iters, int N, int a_tmem, int per_group,
                                                           long long* cycles_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      // a_tmem bit 0: A from TMEM; bit 1: M = 64; bit 2: alternate the accumulator (and TMEM A)
      // between lane offsets 0 and 16 per MMA (two M = 64 products sharing columns)
      const uint32_t idesc = idesc_f16((a_tmem & 2) ? 64 : 128, N, 1, false, false);
      const uint32_t sb = smem_u32(smem);
      for (int it = 0; it < iters; ++it) {
        for (int k = 0; k < per_group; ++k) {
          const uint64_t bd = sdesc_sw128(sb + 32768 + (k & 3) * 32, 16, 1024);
          const uint32_t lo = ((a_tmem & 4) && (k & 1)) ? (16u << 16) : 0u;
          if (a_tmem & 1)
            umma_f16_ts(tmem + lo, tmem + lo + 256 + (k & 7) * 8, bd, idesc, k > 1);
          else
            umma_f16_ss(tmem + lo, sdesc_sw128(sb + (k & 3) * 32, 16, 1024), bd, idesc, k > 1);
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles_out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}
}  // namespace
}  // namespace us

// ---------------------------------------------------------------- MMA pattern probe
// Cycles per iteration of a fixed MMA sequence (one CTA per SM, operands arbitrary):
//   0: 8 SS N=64 (A,B K-major) -> acc0, then 8 SS N=64 (A,B MN-major) -> acc1   [transposed step]
//   1: pattern 0 with every MMA into acc0
//   2: 16 SS N=64 K-major into acc0
//   3: 16 SS N=64 K-major alternating acc0 / acc1 per MMA
//   4: 8 TS N=64 -> acc0, then 4 SS N=128 (B MN-major) -> acc1                  [current step]
//   5: 8 SS N=128 K-major -> acc0, then 8 TS N=128 -> acc1                       [FA4 step]
//   6: 8 SS N=64 (A,B K-major) -> acc0, then 8 SS N=64 (A,B MN-major) -> acc1, A of the second
//      half from two tiles 16 KB apart (the V pair)
namespace us {
namespace {
__global__ void __launch_bounds__(128, 1) mma_pattern_kernel(int iters, int pattern, long long* cycles_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t sb = smem_u32(smem);
      const uint32_t i64k = idesc_f16(128, 64, 1, false, false);
      const uint32_t i64m = idesc_f16(128, 64, 1, true, true);
      const uint32_t i128bm = idesc_f16(128, 128, 1, false, true);
      const uint32_t i128k = idesc_f16(128, 128, 1, false, false);
      for (int it = 0; it < iters; ++it) {
        if (pattern == 0 || pattern == 1 || pattern == 6) {
          for (int k = 0; k < 8; ++k)
            umma_f16_ss(tmem, sdesc_sw128(sb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                        sdesc_sw128(sb + 65536 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024), i64k, k > 0);
          const uint32_t acc = pattern == 1 ? tmem : tmem + 64;
          for (int k = 0; k < 8; ++k) {
            const uint32_t abase = pattern == 6 ? sb + 32768 + (k >> 2) * 16384 + (k & 3) * 2048
                                                : sb + 32768 + k * 2048;
            umma_f16_ss(acc, sdesc_sw128(abase, 8192, 1024), sdesc_sw128(sb + 98304 + k * 2048, 8192, 1024),
                        i64m, pattern == 1 ? 1u : uint32_t(k > 0));
          }
        } else if (pattern == 2 || pattern == 3) {
          for (int k = 0; k < 16; ++k)
            umma_f16_ss(pattern == 3 ? tmem + (k & 1) * 64 : tmem,
                        sdesc_sw128(sb + ((k >> 2) & 1) * 16384 + (k & 3) * 32, 16, 1024),
                        sdesc_sw128(sb + 65536 + ((k >> 2) & 1) * 8192 + (k & 3) * 32, 16, 1024), i64k, k > 1);
        } else if (pattern == 4) {
          for (int k = 0; k < 8; ++k)
            umma_f16_ts(tmem, tmem + 448 + k * 8, sdesc_sw128(sb + 65536 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024),
                        i64k, k > 0);
          for (int k = 0; k < 4; ++k)
            umma_f16_ss(tmem + 64, sdesc_sw128(sb + k * 32, 16, 1024), sdesc_sw128(sb + 98304 + k * 2048, 8192, 1024),
                        i128bm, k > 0);
        } else {
          for (int k = 0; k < 8; ++k)
            umma_f16_ss(tmem, sdesc_sw128(sb + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024),
                        sdesc_sw128(sb + 65536 + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024), i128k, k > 0);
          for (int k = 0; k < 8; ++k)
            umma_f16_ts(tmem + 128, tmem + 384 + k * 8, sdesc_sw128(sb + 98304 + k * 2048, 8192, 1024), i128bm,
                        k > 0);
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles_out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}
}  // namespace
}  // namespace us

extern "C" us_status us_selftest_mma_pattern(int iters, int pattern, int ctas, long long* cycles_out, void* stream) {
  using namespace us;
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(mma_pattern_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_pattern_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(iters, pattern, cycles_out);
  US_LAUNCH_CHECK("us_selftest_mma_pattern");
  return US_OK;
}

extern "C" us_status us_selftest_mma_rate(int iters, int N, int a_tmem, int per_group, int ctas,
                                          long long* cycles_out, void* stream) {
  using namespace us;
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(iters, N, a_tmem, per_group, cycles_out);
  US_LAUNCH_CHECK("us_selftest_mma_rate");
  return US_OK;
}

// ---------------------------------------------------------------- TMEM load bandwidth probe
// Warps 0-3 repeatedly tcgen05.ld 64 fp32 columns of their lane quarter (32x32b.x32 x2)
// and consume them; if mma_n > 0, warp 4 concurrently issues back-to-back
// M=128 x N=mma_n TS-mode MMAs into a disjoint TMEM region. Output: cycles/iteration.
namespace us {
namespace {
__global__ void __launch_bounds__(160, 1) tmem_ld_probe_kernel(int iters, int mma_n, float* sink,
                                                                long long* cycles_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp < 4) {
    float acc = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t v[32], v2[32];
      const uint32_t a = tmem + (uint32_t(warp * 32) << 16) + (it & 1) * 64;
      tmem_ld32(a, v);
      tmem_ld32(a + 32, v2);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += __uint_as_float(v[c]) + __uint_as_float(v2[c]);
    }
    const long long t1 = clock64();
    if (lane == 0 && warp == 0) cycles_out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 128 + threadIdx.x] = acc;
    __syncwarp();
    if (warp == 0 && lane == 0) stop = 1;
  } else if (mma_n > 0) {
    const uint32_t idesc = idesc_f16(128, mma_n, 1, false, false);
    const uint32_t sb = smem_u32(smem);
    int n = 0;
    while (!stop && n < 1000000) {
      if (elect_one()) {
        for (int k = 0; k < 8; ++k) {
          const uint64_t bd = sdesc_sw128(sb + (k & 3) * 32, 16, 1024);
          umma_f16_ts(tmem + 256, tmem + 448 + (k & 7) * 8, bd, idesc, k > 0);
        }
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, n & 1);
      ++n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
}  // namespace
}  // namespace us

extern "C" us_status us_selftest_tmem_ld(int iters, int mma_n, int ctas, float* sink, long long* cycles_out,
                                         void* stream) {
  using namespace us;
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(tmem_ld_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tmem_ld_probe_kernel<<<ctas, 160, smem, static_cast<cudaStream_t>(stream)>>>(iters, mma_n, sink, cycles_out);
  US_LAUNCH_CHECK("us_selftest_tmem_ld");
  return US_OK;
}

// ---------------------------------------------------------------- exp2 throughput probe
// Each thread runs `iters` rounds of 32 independent exp2 evaluations
// (mode 0: MUFU ex2.approx; mode 1: the FMA-pipe cubic of attention.cu;
// mode 2: FFMA2 only, as a pipe-rate reference). Output: cycles per CTA.
namespace us {
namespace {
__device__ __forceinline__ float2 probe_poly2(float2 x) {
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 n = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(n, make_float2(-1.0f, -1.0f), x);
  float2 p = __ffma2_rn(make_float2(0.0551f, 0.0551f), f, make_float2(0.2426f, 0.2426f));
  p = __ffma2_rn(p, f, make_float2(0.6933f, 0.6933f));
  p = __ffma2_rn(p, f, make_float2(0.9999f, 0.9999f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
__global__ void ex2_rate_kernel(int iters, int mode, float* sink, long long* cycles_out) {
  float v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = -0.001f * float(threadIdx.x + c);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = ex2_approx(v[c]) - 1.0f;
    } else if (mode == 1) {
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const float2 p = probe_poly2(make_float2(v[c], v[c + 1]));
        v[c] = p.x - 1.0f;
        v[c + 1] = p.y - 1.0f;
      }
    } else if (mode == 3) {
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        // packed half-precision exp2: one MUFU op for two results (if the pipe allows)
        __half2 h = __floats2half2_rn(v[c], v[c + 1]);
        uint32_t hb = *reinterpret_cast<uint32_t*>(&h), rb;
        asm("ex2.approx.f16x2 %0, %1;" : "=r"(rb) : "r"(hb));
        const float2 r = __half22float2(*reinterpret_cast<__half2*>(&rb));
        v[c] = r.x - 1.0f;
        v[c + 1] = r.y - 1.0f;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const float2 p = __ffma2_rn(make_float2(v[c], v[c + 1]), make_float2(0.999f, 0.999f),
                                    make_float2(0.001f, 0.001f));
        v[c] = p.x;
        v[c + 1] = p.y;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) s += v[c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles_out[blockIdx.x] = t1 - t0;
}
}  // namespace
}  // namespace us

extern "C" us_status us_selftest_ex2_rate(int iters, int mode, int ctas, int threads, float* sink,
                                          long long* cycles_out, void* stream) {
  using namespace us;
  ex2_rate_kernel<<<ctas, threads, 0, static_cast<cudaStream_t>(stream)>>>(iters, mode, sink, cycles_out);
  US_LAUNCH_CHECK("us_selftest_ex2_rate");
  return US_OK;
}

// ---------------------------------------------------------------- softmax-step probe
// The exponential phase of one attention step (attention.cu, 64 key columns per
// thread: row max, FFMA2 scale, 56 MUFU ex2 + 4 cubic pairs, FADD2 row sum, bf16
// pack) on register data, `iters` times back to back, one warp per SMSP (128
// threads) or more. Output: cycles per CTA. Isolates the instruction mix from the
// kernel's TMEM / barrier traffic.
namespace us {
namespace {
__device__ __forceinline__ float2 probe_poly2b(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 n = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(n, make_float2(-1.0f, -1.0f), x);
  float2 p = __ffma2_rn(make_float2(0.0551f, 0.0551f), f, make_float2(0.2426f, 0.2426f));
  p = __ffma2_rn(p, f, make_float2(0.6933f, 0.6933f));
  p = __ffma2_rn(p, f, make_float2(0.9999f, 0.9999f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
__global__ void softmax_probe_kernel(int iters, int mode, uint32_t* sink, long long* cycles_out) {
  // mode bits: 1 = F2FP bf16 packing, 2 = FADD2 row-sum, 4 = row max, 8 = 12.5 % cubic exp2
  float sv[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) sv[c] = 0.01f * float((threadIdx.x * 7 + c * 13) & 63);
  float m_used = 0.f, l = 0.f;
  uint32_t acc_bits = 0;
  const float sl2 = 0.1275f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode & 4) {
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = fmaxf(sv[u], fmaxf(sv[8 + u], sv[16 + u]));
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(sv[24 + u], sv[32 + u]));
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(sv[40 + u], fmaxf(sv[48 + u], sv[56 + u])));
      const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * sl2;
      if (mx > m_used + 8.f) m_used = mx;
    }
    const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_used, -m_used);
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t packed[32];
#pragma unroll
    for (int c = 0; c < 64; c += 2) {
      const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
      float2 p;
      if ((mode & 8) && c >= 56) {
        p = probe_poly2b(xx);
      } else {
        p.x = ex2_approx(xx.x);
        p.y = ex2_approx(xx.y);
      }
      if (mode & 2) acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
      packed[c >> 1] = (mode & 1) ? pack_bf16(p.x, p.y) : (__float_as_uint(p.x) ^ __float_as_uint(p.y));
    }
    const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
    l += s2.x + s2.y;
#pragma unroll
    for (int w = 16; w > 0; w >>= 1)
#pragma unroll
      for (int c = 0; c < w; ++c) packed[c] ^= packed[c + w];
    acc_bits ^= packed[0];
    m_used += 1e-7f;
  }
  __syncthreads();
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc_bits ^ __float_as_uint(l);
  if (threadIdx.x == 0) cycles_out[blockIdx.x] = t1 - t0;
}
}  // namespace
}  // namespace us

extern "C" us_status us_selftest_softmax_probe(int iters, int mode, int ctas, int threads, uint32_t* sink,
                                               long long* cycles_out, void* stream) {
  using namespace us;
  softmax_probe_kernel<<<ctas, threads, 0, static_cast<cudaStream_t>(stream)>>>(iters, mode, sink, cycles_out);
  US_LAUNCH_CHECK("us_selftest_softmax_probe");
  return US_OK;
}

// ---------------------------------------------------------------- M = 64 accumulator layout probe
// One M = 64, N = 64, K = 128 kind::f16 MMA (A rows 0-63 and B both K-major SW128 in smem,
// written by threads) with the accumulator address at TMEM lane offset `lane_off`; TMEM
// columns [0, 64) of all 128 lanes are first filled with a sentinel and read back after, so
// the host sees which lanes the 64 result rows land in (D_out [128 lanes][64 cols] f32).
namespace us {
namespace {
// ts = 1: A from TMEM instead — A2 [128][128] bf16 rows 64 r + ... : rows 0-63 of A at lanes
// (16 q + r) of quarter q (offset 0), rows 64-127 at lanes 16 + (16 q + r) (offset 16), in
// TMEM columns [64, 128); two MMAs: D at offset 0 with A offset 0, D at offset 16 (columns
// [0, 64)) with A offset 16 — then D_out holds both results.
__global__ void __launch_bounds__(128, 1)
    m64_probe_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, int lane_off, float* D_out,
                     int ts) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // [kc][64 rows][128 B]
  uint8_t* sB = smem + 64 * 128 * 2;  // [kc][64 rows][128 B]
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base_sh;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  {
    uint32_t v[16];
    for (int t = 0; t < 16; ++t) v[t] = __float_as_uint(12345.0f);
    for (int c0 = 0; c0 < 64; c0 += 16) tmem_st16(tmem + lane_base + c0, v);
    tmem_st_wait();
  }
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    for (int kc = 0; kc < 2; ++kc)
      for (int ch = 0; ch < 8; ++ch) {
        *reinterpret_cast<uint4*>(sA + kc * 64 * 128 + sw128_offset(r, ch)) =
            *reinterpret_cast<const uint4*>(A + r * 128 + kc * 64 + ch * 8);
        *reinterpret_cast<uint4*>(sB + kc * 64 * 128 + sw128_offset(r, ch)) =
            *reinterpret_cast<const uint4*>(B + r * 128 + kc * 64 + ch * 8);
      }
  }
  if (ts == 1 || ts >= 2) {
    // lane 32 q + i holds A row (i < 16 ? 16 q + i : 64 + 16 q + (i - 16)); 2 bf16 per column
    const int i = lane;
    const int arow = i < 16 ? 16 * warp + i : 64 + 16 * warp + (i - 16);
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t v[16];
      for (int t = 0; t < 16; ++t)
        v[t] = uint32_t(A[arow * 128 + 2 * (c0 + t)]) | (uint32_t(A[arow * 128 + 2 * (c0 + t) + 1]) << 16);
      tmem_st16(tmem + lane_base + 64 + c0, v);
    }
    tmem_st_wait();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_f16(64, 64, 1, false, false);
      if (ts == 0) {
        for (int k = 0; k < 8; ++k) {
          const int kc = k / 4, ks = k % 4;
          const uint64_t ad = sdesc_sw128(smem_u32(sA + kc * 64 * 128 + ks * 32), 16, 1024);
          const uint64_t bd = sdesc_sw128(smem_u32(sB + kc * 64 * 128 + ks * 32), 16, 1024);
          umma_f16_ss(tmem + (uint32_t(lane_off) << 16), ad, bd, idesc, k > 0);
        }
      } else {
        for (int off = 0; off < 32; off += 16)
          for (int k = 0; k < 8; ++k) {
            const int kc = k / 4, ks = k % 4;
            const uint64_t bd = sdesc_sw128(smem_u32(sB + kc * 64 * 128 + ks * 32), 16, 1024);
            umma_f16_ts(tmem + (uint32_t(off) << 16), tmem + (uint32_t(off) << 16) + 64 + k * 8, bd, idesc, k > 0);
          }
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  if (ts >= 2) {
    // 16x32bx2 read of the accumulator at lane offset (ts - 2) * 16 of each quarter:
    // D_out[warp][lane][32] = what thread `lane` of warp `warp` receives
    uint32_t v[32];
    tmem_ld_16x32bx2_x32<32>(tmem + lane_base + (uint32_t((ts - 2) * 16) << 16), v);
    tmem_ld_wait();
    for (int t = 0; t < 32; ++t) D_out[row * 64 + t] = __uint_as_float(v[t]);
  } else {
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + c0, v);
      tmem_ld_wait();
      for (int t = 0; t < 16; ++t) D_out[row * 64 + c0 + t] = __uint_as_float(v[t]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 128);
}
}  // namespace
}  // namespace us

extern "C" us_status us_selftest_m64_layout(const void* A, const void* B, int lane_off, int ts, float* D_out,
                                           void* stream) {
  using namespace us;
  const size_t smem = 32 * 1024 + 1024;
  m64_probe_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(A), static_cast<const uint16_t*>(B), lane_off, D_out, ts);
  US_LAUNCH_CHECK("us_selftest_m64_layout");
  return US_OK;
}
