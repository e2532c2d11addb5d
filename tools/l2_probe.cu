// l2_probe.cu — L2 -> SMEM bulk-copy throughput (calibration tool, not product code).
// Each CTA streams `chunk`-byte tiles from pseudo-random chunk-aligned offsets of a
// `region`-byte buffer into an NS-stage SMEM ring (1-D cp.async.bulk, mbarrier
// complete_tx), the way attn_kernel streams selected K/V tiles. Prints GB/s for
// several region sizes (L2-resident vs DRAM) and CTA counts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_tmp_l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void __launch_bounds__(64) probe(const uint8_t* __restrict__ buf, long long region, int chunk,
                                            int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NS];
  const long long nchunks = region / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1);
  auto issue = [&](int t) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const long long c = (long long)(x % (unsigned long long)nchunks);
    const int s = t % NS;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + (size_t)s * chunk)), "l"(buf + c * chunk), "r"(chunk), "r"(su32(&full[s]))
                 : "memory");
  };
  for (int t = 0; t < NS && t < iters; ++t) issue(t);
  unsigned long long acc = 0;
  for (int t = 0; t < iters; ++t) {
    const int s = t % NS;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                   : "=r"(ok) : "r"(su32(&full[s])), "r"((t / NS) & 1) : "memory");
    acc += sm[(size_t)s * chunk + (t & 127)];
    if (t + NS < iters) issue(t + NS);
  }
  if (acc == 0xFFFFFFFFull) *sink = acc;
}

int main() {
  const long long maxregion = 1ll << 30;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, maxregion);
  cudaMemset(buf, 1, maxregion);
  cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(probe<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long regions[] = {16ll << 20, 64ll << 20, 96ll << 20, 1ll << 30};
  const int chunks[] = {16384, 32768};
  const int ctas_per_sm[] = {1, 2};
  for (long long region : regions)
    for (int chunk : chunks)
      for (int cps : ctas_per_sm) {
        const int grid = 148 * cps, iters = 4000;
        const int smem = 6 * chunk;
        if (smem * cps > 220 * 1024) continue;
        probe<6><<<grid, 64, smem>>>(buf, region, chunk, 200, sink);
        cudaEventRecord(a);
        probe<6><<<grid, 64, smem>>>(buf, region, chunk, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = double(grid) * iters * chunk;
        printf("region %5lld MB chunk %5d B ctas/SM %d stages 6: %8.1f GB/s\n", region >> 20, chunk, cps,
               bytes / ms / 1e6);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
