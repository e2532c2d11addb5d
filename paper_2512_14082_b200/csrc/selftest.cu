// selftest.cu — single-tile tcgen05 checks of every operand path the hot
// kernels rely on (exported as us_selftest_umma, exercised by tests/test_gpu_selftest.py):
//   mode 0: A K-major (TMA), B K-major (TMA)            D = A * B^T   (proxy Q.K^T, attention S)
//   mode 1: A K-major (TMA), B MN-major (TMA)           D = A * B     (attention P.V with V row-major)
//   mode 2: A in TMEM (tcgen05.st), B K-major (TMA)     D = A * B^T   (TS path)
//   mode 3: A written by threads into swizzled smem, B MN-major: the attention P.V path.
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

  const bool b_mn = (mode == 1 || mode == 3);
  // ---- operand staging
  if (threadIdx.x == 0) {
    uint32_t bytes = N * kK * 2;
    if (mode <= 1) bytes += kM * kK * 2;
    mbar_arrive_expect_tx(&bar_tma, bytes);
    if (mode <= 1)
      for (int kc = 0; kc < 2; ++kc) tma_load_2d(sA + kc * kM * 128, &tmA, &bar_tma, kc * 64, 0);
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
      const uint32_t idesc = idesc_f16(kM, N, bf16 ? 1 : 0, false, b_mn);
      for (int k = 0; k < kK / 16; ++k) {
        const int kc = k / 4, ks = k % 4;
        uint64_t bdesc;
        if (!b_mn)
          bdesc = sdesc_sw128(smem_u32(sB + kc * N * 128 + ks * 32), 16, 1024);
        else
          bdesc = sdesc_sw128(smem_u32(sB + k * 16 * 128), kK * 128, 1024);
        if (mode == 2) {
          umma_f16_ts(tmem, tmem + 128 + k * 8, bdesc, idesc, k > 0);
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
  if (mode < 0 || mode > 3 || (N != 64 && N != 128)) {
    set_error("us_selftest_umma: bad mode/N");
    return US_ERR_INVALID_ARGUMENT;
  }
  CUtensorMap tmA{}, tmB{};
  us_status s = make_tmap_2d_16b(&tmA, A, kM, kK, kM, 64, bf16);
  if (s != US_OK) return s;
  const bool b_mn = (mode == 1 || mode == 3);
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
