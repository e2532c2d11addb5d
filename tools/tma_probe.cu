// tma_probe.cu — L2 -> SMEM throughput of 16 KB K/V tiles loaded the way the attention
// kernels load them (calibration tool, not product code). Each CTA (one per SM) streams
// tiles of 64 rows x 256 B (64 keys x d = 128 bf16) from random 64-row-aligned offsets of
// one region (a KV head's K+V: 64 MB) into an NS-stage SMEM ring:
//   mode 0: one 3-D rows-chunked tensor TMA per tile (SWIZZLE_128B; attention*.cu)
//   mode 1: two 2-D tensor TMAs per tile (64 cols x 64 rows each, SWIZZLE_128B)
//   mode 2: one 1-D cp.async.bulk of the tile's 16 contiguous KB (no swizzle)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tmp_tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) probe(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m2,
                                            const uint8_t* __restrict__ buf, long long rows, int mode, int ns,
                                            int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smb[];
  __shared__ uint64_t fullb[64];
  // issuing warp w (lane 0): its own ns-stage ring and barriers
  const int w = threadIdx.x >> 5;
  uint8_t* sm = smb + (size_t)w * ns * 16384;
  uint64_t* full = fullb + w * ns;
  if ((threadIdx.x & 31) == 0) {
    for (int s = 0; s < ns; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if ((threadIdx.x & 31) != 0) return;
  const long long tiles = rows / 64;
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * 8 + w + 1);
  auto issue = [&](int t) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    // mode >= 3: power-of-two tile count, no 64-bit modulo (issue-loop cost check)
    const int row = mode >= 3 ? int((uint32_t(x >> 20) & uint32_t(tiles - 1)) * 64)
                              : int((x % (unsigned long long)tiles) * 64);
    const int s = t % ns;
    uint8_t* dst = sm + (size_t)s * 16384;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384) : "memory");
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su32(dst)), "l"(&m3), "r"(su32(&full[s])), "r"(0), "r"(row), "r"(0) : "memory");
    } else if (mode == 1) {
      for (int c = 0; c < 2; ++c)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(dst + c * 8192)), "l"(&m2), "r"(su32(&full[s])), "r"(c * 64), "r"(row) : "memory");
    } else if (mode == 4) {  // two 8 KB halves: per-instruction cost
      for (int c = 0; c < 2; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(dst + c * 8192)), "l"(buf + (size_t)row * 256 + c * 8192), "r"(8192), "r"(su32(&full[s]))
                     : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(dst)), "l"(buf + (size_t)row * 256), "r"(16384), "r"(su32(&full[s])) : "memory");
    }
  };
  for (int t = 0; t < ns && t < iters; ++t) issue(t);
  unsigned long long acc = 0;
  for (int t = 0; t < iters; ++t) {
    const int s = t % ns;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                   : "=r"(ok) : "r"(su32(&full[s])), "r"((t / ns) & 1) : "memory");
    acc += sm[(size_t)s * 16384 + (t & 127)];
    if (t + ns < iters) issue(t + ns);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

int main() {
  const long long region = 64ll << 20, rows = region / 256;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, region);
  cudaMemset(buf, 1, region);
  cudaMalloc(&sink, 8);
  CUtensorMap m3, m2;
  {
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
    cuuint64_t strides[2] = {256, 128};
    cuuint32_t box[3] = {64, 64, 2}, estr[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode 3d failed %d\n", int(r));
  }
  {
    cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 64}, estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode 2d failed %d\n", int(r));
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names2[5] = {"3-D tensor (attention)", "2 x 2-D tensor", "1-D bulk", "1-D bulk, no modulo",
                           "2 x 8 KB bulk, no modulo"};
  // issuers per SM: c CTAs per SM x p issuing warps per CTA, ns stages each
  for (int mode : {0, 3})
    for (int c : {1, 2})
      for (int p : {1, 2, 4})
        for (int ns : {2, 4}) {
          const int grid = 148 * c, iters = 2000;
          if (c * p * ns * 16384 > 200 * 1024) continue;
          probe<<<grid, 32 * p, p * ns * 16384>>>(m3, m2, buf, rows, mode, ns, 100, sink);
          cudaEventRecord(a);
          probe<<<grid, 32 * p, p * ns * 16384>>>(m3, m2, buf, rows, mode, ns, iters, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double bytes = double(grid) * p * iters * 16384;
          printf("%-24s CTAs/SM %d x issuing warps %d, stages %d each: %8.1f GB/s  %5.1f B/clk/SM\n", names2[mode],
                 c, p, ns, bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / 1.9e9);
        }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
