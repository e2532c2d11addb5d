// lastblock.cu — FlexPrefill-style last-block probe on the GPU (
// reference last_block_probe_scores, baselines.cpp:54-87).
//
// The last S query rows of every head attend (causally) to all keys; each key
// block's column mass colmass(j) = sum over those rows of the softmax mass of
// the block's keys becomes the score of (i, j) for every causal row i >= j.
// The work is a skinny 64 x L x d product per head, so it runs on the CUDA
// cores (fp32 FMA of exact bf16 products), thread = key, the 64 query rows in
// shared memory:
//   lb_stats_kernel:    per 256-key chunk and query row, max and sum of 2^(x - max)
//   lb_lse_kernel:      per query row, the row LSE over all chunks (fixed order)
//   lb_colmass_kernel:  recompute the logits, p = 2^(x - lse), per-key sum over the
//                       rows, per-block sum -> colmass (fixed order)
//   lb_broadcast_kernel: scores[i][j] = colmass[j] for j <= i
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

constexpr int kRowsLB = 64;   // S (GPU path block size)
constexpr int kChunk = 256;   // keys per CTA

template <int D>
__device__ __forceinline__ void load_q_rows(const LastBlockArgs& a, int plane, float (*qs)[D]) {
  const uint16_t* q = a.Q + ((long long)plane * a.L + (long long)(a.N - 1) * kRowsLB) * D;
  for (int e = threadIdx.x; e < kRowsLB * D; e += blockDim.x)
    qs[e / D][e % D] = __uint_as_float(uint32_t(q[e]) << 16);
}

template <int D>
__device__ __forceinline__ void key_logits(const LastBlockArgs& a, int plane, int key, float (*qs)[D],
                                           float (&lg)[kRowsLB]) {
  const int b = plane / a.H, h = plane % a.H;
  const uint16_t* k = a.K + (((long long)b * a.H_kv + h / (a.H / a.H_kv)) * a.L + key) * D;
  float kv[D];
#pragma unroll
  for (int c = 0; c < D; c += 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(k + c);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      kv[c + 2 * u] = __uint_as_float(w[u] << 16);
      kv[c + 2 * u + 1] = __uint_as_float(w[u] & 0xFFFF0000u);
    }
  }
  const int first_row = (a.N - 1) * kRowsLB;
#pragma unroll 4
  for (int r = 0; r < kRowsLB; ++r) {
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) acc = fmaf(qs[r][c], kv[c], acc);
    lg[r] = key <= first_row + r ? acc * a.scale_log2 : -INFINITY;  // causal: live = first_row + r + 1
  }
}

template <int D>
__global__ void __launch_bounds__(kChunk) lb_stats_kernel(const LastBlockArgs a) {
  __shared__ float qs[kRowsLB][D];
  __shared__ float red[kRowsLB][kChunk / 32];
  const int plane = blockIdx.y, chunk = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  load_q_rows<D>(a, plane, qs);
  __syncthreads();
  float lg[kRowsLB];
  key_logits<D>(a, plane, chunk * kChunk + threadIdx.x, qs, lg);
  // chunk max per row
#pragma unroll 4
  for (int r = 0; r < kRowsLB; ++r) {
    float m = lg[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[r][warp] = m;
  }
  __syncthreads();
  __shared__ float cmax[kRowsLB];
  if (threadIdx.x < kRowsLB) {
    float m = red[threadIdx.x][0];
    for (int w = 1; w < kChunk / 32; ++w) m = fmaxf(m, red[threadIdx.x][w]);
    cmax[threadIdx.x] = m;
  }
  __syncthreads();
  // chunk sum of 2^(x - chunk max) per row, fixed tree (red is reused: every
  // thread has read the maxima above)
#pragma unroll 4
  for (int r = 0; r < kRowsLB; ++r) {
    float s = cmax[r] == -INFINITY ? 0.f : ex2_approx(lg[r] - cmax[r]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[r][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < kRowsLB) {
    float s = 0.f;
    for (int w = 0; w < kChunk / 32; ++w) s += red[threadIdx.x][w];
    const long long o = ((long long)plane * gridDim.x + chunk) * kRowsLB + threadIdx.x;
    a.cmax[o] = cmax[threadIdx.x];
    a.csum[o] = s;
  }
}

__global__ void lb_lse_kernel(const LastBlockArgs a, int nchunks) {
  const int plane = blockIdx.x, r = threadIdx.x;
  float m = -INFINITY;
  for (int c = 0; c < nchunks; ++c) m = fmaxf(m, a.cmax[((long long)plane * nchunks + c) * kRowsLB + r]);
  float l = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const long long o = ((long long)plane * nchunks + c) * kRowsLB + r;
    if (a.cmax[o] != -INFINITY) l += a.csum[o] * ex2_approx(a.cmax[o] - m);
  }
  a.lse2[(long long)plane * kRowsLB + r] = m + __log2f(l);
}

template <int D>
__global__ void __launch_bounds__(kChunk) lb_colmass_kernel(const LastBlockArgs a) {
  __shared__ float qs[kRowsLB][D];
  __shared__ float lse[kRowsLB];
  __shared__ float wsum[kChunk / 32];
  const int plane = blockIdx.y, chunk = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  load_q_rows<D>(a, plane, qs);
  if (threadIdx.x < kRowsLB) lse[threadIdx.x] = a.lse2[(long long)plane * kRowsLB + threadIdx.x];
  __syncthreads();
  float lg[kRowsLB];
  key_logits<D>(a, plane, chunk * kChunk + threadIdx.x, qs, lg);
  float col = 0.f;  // this key's mass over the 64 rows, row order
#pragma unroll
  for (int r = 0; r < kRowsLB; ++r) col += lg[r] == -INFINITY ? 0.f : ex2_approx(lg[r] - lse[r]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) col += __shfl_xor_sync(0xffffffffu, col, o);
  if (lane == 0) wsum[warp] = col;
  __syncthreads();
  // a 64-key block = 2 warps
  if (threadIdx.x < kChunk / kRowsLB) {
    const int j = chunk * (kChunk / kRowsLB) + threadIdx.x;
    a.colmass[(long long)plane * a.N + j] = wsum[2 * threadIdx.x] + wsum[2 * threadIdx.x + 1];
  }
}

__global__ void lb_broadcast_kernel(const LastBlockArgs a) {
  const int plane = blockIdx.y, i = blockIdx.x;
  float* out = a.scores + ((long long)plane * a.N + i) * a.N;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) out[j] = a.colmass[(long long)plane * a.N + j];
}

template <int D>
us_status launch_lb_t(const LastBlockArgs& a, cudaStream_t st) {
  const int nchunks = a.L / kChunk;
  const dim3 grid(nchunks, a.B * a.H);
  lb_stats_kernel<D><<<grid, kChunk, 0, st>>>(a);
  US_LAUNCH_CHECK("lb_stats_kernel");
  lb_lse_kernel<<<a.B * a.H, kRowsLB, 0, st>>>(a, nchunks);
  US_LAUNCH_CHECK("lb_lse_kernel");
  lb_colmass_kernel<D><<<grid, kChunk, 0, st>>>(a);
  US_LAUNCH_CHECK("lb_colmass_kernel");
  lb_broadcast_kernel<<<dim3(a.N, a.B * a.H), 256, 0, st>>>(a);
  US_LAUNCH_CHECK("lb_broadcast_kernel");
  return US_OK;
}

}  // namespace

us_status launch_last_block_probe(const LastBlockArgs& a, cudaStream_t st) {
  if (a.N * kRowsLB != a.L) {
    set_error("select_blocks: the last-block probe runs at block size S = 64 on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.L % kChunk != 0) {
    set_error("select_blocks: the last-block probe needs L divisible by 256 on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_lb_t<128>(a, st);
  if (a.D == 64) return launch_lb_t<64>(a, st);
  set_error("select_blocks: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
