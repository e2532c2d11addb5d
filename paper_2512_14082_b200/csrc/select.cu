// select.cu — per-row Top-P / top-k block selection.
//
// Reference semantics (selection.cpp:11-48): order = descending score, ties by
// ascending index (stable_sort); total = fp64 sum in that order; walk the order
// accumulating fp64 cum and stop at the first element with cum >= P * total
// (inclusive). All-zero rows select the diagonal; P >= 1 selects the prefix.
// top-k: the first min(k, i+1) entries of the same order.
//
// GPU algorithm (one warp per row, scores as f32 bit patterns in registers —
// non-negative floats order like their unsigned bits):
//   1. total = fp64 warp sum (fixed tree).
//   2. bisection over the value bits for v* = the largest value whose tail mass
//      G(v*) = sum_{x >= v*} x reaches T = P * total, with fp32 tail sums (cheap;
//      a candidate that fp32 rounding put on the wrong side of T is caught by the
//      certification below); top-k: bisection on the tail count.
//   3. A = sum_{x > v*} x; walk the ties of v* in index order: cum = A + v*,
//      A + 2v*, ... until cum >= T — exactly the reference walk across the
//      boundary group.
//   4. Certification: the reference sums sequentially in sorted order; our sums
//      use a different (tree) order. Two fp64 summation orders of n
//      non-negative terms differ by at most 2 n u total (u = 2^-53). Every
//      comparison against T is therefore accepted only when its margin exceeds
//      eps = 4 n u total; otherwise the row goes to select_fallback_kernel,
//      which sorts the row and reproduces the reference's sequential fp64 walk
//      verbatim. Result: masks identical to the reference rule applied to the
//      same f32 scores, for every row (tests/test_gpu_select.py pins this).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"
#include "proxy_score.cuh"

namespace us {
namespace {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One row on one warp; NPL = 32-element chunks per lane held in registers (the
// caller picks the smallest instantiation that covers the row's causal prefix,
// so short rows do not pay for the longest one's predicated-off work).
template <int NPL>
__device__ __forceinline__ void select_row(const SelectArgs& a, long long row, int lane, uint32_t lt_mask) {
  {
    const int i = int(row % a.N);
    const int n = i + 1;
    const float* src = a.scores + row * a.N;
    uint32_t bits[NPL];
    bool bad = false, nonfinite = false;
    double part = 0.0;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      bits[k] = 0;
      const int idx = k * 32 + lane;
      if (k * 32 < n && idx < n) {
        float f = __ldg(src + idx);
        if (!(f >= 0.f)) {
          bad = true;
          f = 0.f;
        }
        if (f == 0.f) f = 0.f;  // -0 -> +0
        if (isinf(f)) nonfinite = true;
        bits[k] = __float_as_uint(f);
        part += double(f);
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, 1u);
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    const double total = warp_sum_f64(part);

    uint32_t bstar = 0;     // threshold value bits
    int ties_needed = 0;    // how many elements equal to v* (lowest index first) are taken
    int mode = 0;           // 0: threshold rule, 1: all, 2: diagonal only
    double cum = 0.0;
    bool certified = true;
    if (a.select_mode == US_SELECT_TOP_K) {
      const int kk = min(a.top_k, n);
      for (int bit = 30; bit >= 0; --bit) {
        const uint32_t cand = bstar | (1u << bit);
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < NPL; ++k)
          if (k * 32 < n) cnt += (k * 32 + lane < n && bits[k] >= cand) ? 1 : 0;
        if (int(__reduce_add_sync(0xffffffffu, unsigned(cnt))) >= kk) bstar = cand;
      }
      int gt = 0;
#pragma unroll
      for (int k = 0; k < NPL; ++k)
        if (k * 32 < n) gt += (k * 32 + lane < n && bits[k] > bstar) ? 1 : 0;
      ties_needed = kk - warp_sum_i32(gt);
    } else if (!(total > 0.0)) {
      mode = 2;
    } else if (a.P >= 1.0) {
      mode = 1;
    } else if (nonfinite) {
      certified = false;  // let the exact path handle inf arithmetic
      mode = 1;
    } else {
      const double T = a.P * total;
      // (a) candidate v* by bisection over the value bits with fp32 tail sums
      //     (4 independent accumulators per lane, fixed shuffle tree) — cheap, but
      //     only approximately ordered against T;
      const float Tf = float(T);
      uint32_t mx = 0;
#pragma unroll
      for (int k = 0; k < NPL; ++k) mx = max(mx, bits[k]);
      mx = __reduce_max_sync(0xffffffffu, mx);
      const int top = 31 - __clz(mx | 1u);
      for (int bit = top; bit >= 0; --bit) {
        const uint32_t cand = bstar | (1u << bit);
        float g8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < NPL; ++k)
          if (k * 32 < n) g8[k & 7] += bits[k] >= cand ? __uint_as_float(bits[k]) : 0.f;
        const float g = ((g8[0] + g8[1]) + (g8[2] + g8[3])) + ((g8[4] + g8[5]) + (g8[6] + g8[7]));
        if (warp_sum_f32(g) >= Tf) bstar = cand;
      }
      // (b) exact fp64 boundary walk + certification (a wrong candidate from (a)
      //     fails certification and goes to the verbatim reference walk).
      double A = 0.0;
      int E = 0;
#pragma unroll
      for (int k = 0; k < NPL; ++k) {
        if (k * 32 < n && k * 32 + lane < n) {
          if (bits[k] > bstar) A += double(__uint_as_float(bits[k]));
          if (bits[k] == bstar) ++E;
        }
      }
      A = warp_sum_f64(A);
      E = warp_sum_i32(E);
      const double eps = 4.0 * double(n) * 0x1p-53 * total;
      const double vstar = double(__uint_as_float(bstar));
      cum = A;
      certified = (T - cum) > eps;
      int c = 0;
      while (c < E) {
        cum += vstar;
        ++c;
        if (cum >= T) break;
        certified = certified && (T - cum) > eps;
      }
      certified = certified && (cum >= T) && (cum - T) > eps;
      ties_needed = c;
    }

    // ---- emit selection
    int tie_base = 0, sel_count = 0;
    double sel_mass = 0.0;
    uint32_t* mrow = a.mask_bits + row * a.W;
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      if (k >= a.W) break;
      const int idx = k * 32 + lane;
      const bool valid = idx < n;
      bool sel;
      if (mode == 1) {
        sel = valid;
      } else if (mode == 2) {
        sel = idx == n - 1;
      } else {
        const bool tie = valid && bits[k] == bstar;
        const uint32_t tmask = __ballot_sync(0xffffffffu, tie);
        const int rank = tie_base + __popc(tmask & lt_mask);
        tie_base += __popc(tmask);
        sel = valid && (bits[k] > bstar || (tie && rank < ties_needed));
      }
      const uint32_t word = __ballot_sync(0xffffffffu, sel);
      if (lane == 0) mrow[k] = word;
      if (a.indices && sel) a.indices[row * a.N + sel_count + __popc(word & lt_mask)] = int16_t(idx);
      if (sel) sel_mass += double(__uint_as_float(bits[k]));
      sel_count += __popc(word);
    }
    for (int k = NPL + lane; k < a.W; k += 32) mrow[k] = 0u;  // (never taken when NPL*32 >= N)
    double cov;
    if (a.select_mode == US_SELECT_TOP_K) {
      const double m = warp_sum_f64(sel_mass);
      cov = total > 0.0 ? m / total : 1.0;
    } else {
      cov = mode == 0 ? cum / total : 1.0;
    }
    if (lane == 0) {
      if (a.counts) a.counts[row] = sel_count;
      if (a.coverage) a.coverage[row] = cov;
      if (!certified) a.fb_rows[atomicAdd(a.fb_count, 1)] = int32_t(row);
    }
  }
}

template <int NPL>
__global__ void __launch_bounds__(256, 2) select_kernel(SelectArgs a) {
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  // eighths of the longest row (quarters / halves / whole for short N)
  constexpr int E = NPL >= 8 ? NPL / 8 : 1;
  for (long long row = (long long)blockIdx.x * wpc + (threadIdx.x >> 5); row < a.rows;
       row += (long long)gridDim.x * wpc) {
    const int n = int(row % a.N) + 1;
    if (NPL < 8) {
      if (n <= 32 * (NPL >= 4 ? NPL / 4 : 1)) select_row<(NPL >= 4 ? NPL / 4 : 1)>(a, row, lane, lt_mask);
      else if (n <= 32 * (NPL >= 2 ? NPL / 2 : 1)) select_row<(NPL >= 2 ? NPL / 2 : 1)>(a, row, lane, lt_mask);
      else select_row<NPL>(a, row, lane, lt_mask);
    } else if (n <= 32 * E) select_row<E>(a, row, lane, lt_mask);
    else if (n <= 64 * E) select_row<2 * E>(a, row, lane, lt_mask);
    else if (n <= 96 * E) select_row<3 * E>(a, row, lane, lt_mask);
    else if (n <= 128 * E) select_row<4 * E>(a, row, lane, lt_mask);
    else if (n <= 160 * E) select_row<5 * E>(a, row, lane, lt_mask);
    else if (n <= 192 * E) select_row<6 * E>(a, row, lane, lt_mask);
    else if (n <= 224 * E) select_row<7 * E>(a, row, lane, lt_mask);
    else select_row<NPL>(a, row, lane, lt_mask);
  }
}

// Exact reference walk for uncertified rows: bitonic sort of (value desc,
// index asc) keys in smem, then one thread sums in sorted order in fp64
// (selection.cpp:25-46 verbatim).
constexpr int kFbMaxN = 4096;
__global__ void __launch_bounds__(256) select_fallback_kernel(SelectArgs a) {
  __shared__ unsigned long long keys[kFbMaxN];
  __shared__ uint8_t flag[kFbMaxN];
  __shared__ int sh_k;
  __shared__ double sh_cov;
  const int count = *a.fb_count;
  for (int e = blockIdx.x; e < count; e += gridDim.x) {
    const long long row = a.fb_rows[e];
    const int i = int(row % a.N), n = i + 1;
    const float* src = a.scores + row * a.N;
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int t = threadIdx.x; t < n2; t += blockDim.x) {
      if (t < n) {
        float f = src[t];
        if (!(f >= 0.f) || f == 0.f) f = 0.f;
        keys[t] = ((unsigned long long)(~__float_as_uint(f)) << 32) | unsigned(t);
      } else {
        keys[t] = ~0ull;
      }
      flag[t] = 0;
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < n2; t += blockDim.x) {
          const int p = t ^ j;
          if (p > t) {
            const unsigned long long x = keys[t], y = keys[p];
            const bool up = (t & k) == 0;
            if ((x > y) == up) {
              keys[t] = y;
              keys[p] = x;
            }
          }
        }
        __syncthreads();
      }
    if (threadIdx.x == 0) {
      auto val = [&](int t) { return double(__uint_as_float(~unsigned(keys[t] >> 32))); };
      double total = 0.0;
      for (int t = 0; t < n; ++t) total += val(t);
      int ksel;
      double cov = 1.0;
      if (total <= 0.0) {
        ksel = -1;  // diagonal only
      } else if (a.P >= 1.0) {
        ksel = n;
      } else {
        double cum = 0.0;
        ksel = 0;
        for (int t = 0; t < n; ++t) {
          ++ksel;
          cum += val(t);
          if (cum >= a.P * total) break;
        }
        cov = cum / total;
      }
      sh_k = ksel;
      sh_cov = cov;
    }
    __syncthreads();
    const int ksel = sh_k;
    if (ksel < 0) {
      if (threadIdx.x == 0) flag[n - 1] = 1;
    } else {
      for (int t = threadIdx.x; t < ksel; t += blockDim.x) flag[unsigned(keys[t] & 0xFFFFFFFFu)] = 1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int base = 0;
      for (int w = 0; w < a.W; ++w) {
        const int idx = w * 32 + lane;
        const bool sel = idx < n && flag[idx];
        const uint32_t word = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) a.mask_bits[row * a.W + w] = word;
        if (a.indices && sel) a.indices[row * a.N + base + __popc(word & ((1u << lane) - 1u))] = int16_t(idx);
        base += __popc(word);
      }
      if (lane == 0) {
        if (a.counts) a.counts[row] = base;
        if (a.coverage) a.coverage[row] = sh_cov;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- fused finalize + selection
// One CTA (256 threads) per (plane, query block) row, rows heaviest first in a
// grid-stride loop. The row's scores are built in shared memory from the proxy's
// slot partials (the block_aggregate of proxy.cpp:48-72, bit-identical to the
// standalone finalize), never round-tripping through HBM. Selection:
//   Top-P: radix descent over the value bits (11 + 11 + 9 bits, float mass
//          histograms in smem) finds the candidate threshold v* with
//          G(v*) = sum_{x >= v*} x >= T = P * total; then the exact fp64 boundary
//          walk and the 4 n u total certification of select_row; an uncertified row
//          goes to the exact sorted walk (select_fallback_fused_kernel).
//   top-k: the same descent on counts (exact), ties by ascending index.
constexpr int kFusedThreads = 128;
constexpr int kFusedWarps = kFusedThreads / 32;
constexpr int kFusedMaxW = kFbMaxN / 32;
constexpr int kRadixBins = 256;
constexpr int kMaxFacTiles = 256;  // c = 8 fast path: key tiles per row (L/8/128 <= 256 at L <= 256K)
// calibration knobs (tools/build_src_variant.sh): scores per thread in flight in the score
// phase, resident CTAs per SM asked of ptxas, warp-aggregated histogram updates
#ifndef US_SEL_INFLIGHT
#define US_SEL_INFLIGHT 4
#endif
// (US_SEL_MINB unset: plain __launch_bounds__(128) — asking for 1 block per SM lets ptxas
// take 103 registers instead of 56, halving the resident CTAs: 1.35 -> 1.8 ms at C3)
#ifdef US_SEL_MINB
#define US_SEL_LAUNCH_BOUNDS __launch_bounds__(kFusedThreads, US_SEL_MINB)
#else
#define US_SEL_LAUNCH_BOUNDS __launch_bounds__(kFusedThreads)
#endif
#ifndef US_SEL_AGG
#define US_SEL_AGG 0
#endif
// grid 32 x 148 CTAs without the L2 prefetch of each CTA's next row: -4.5 % at C3 vs
// 16 x 148 with it (profiles/r02k; the 9 resident CTAs per SM already keep enough loads
// in flight, and the prefetched rows of 2 x 1332 CTAs overflow the L2)
#ifndef US_SEL_GRID_PER_SM
#define US_SEL_GRID_PER_SM 32
#endif
#ifndef US_SEL_PREFETCH
#define US_SEL_PREFETCH 0
#endif

__device__ __forceinline__ double block_sum_f64(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum_f64(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kFusedWarps; ++w) t += sh[w];  // fixed order
  return t;
}
__device__ __forceinline__ int block_sum_i32(int v, int* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum_i32(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < kFusedWarps; ++w) t += sh[w];
  return t;
}
// exclusive prefix over W <= 128 per-word counts (warp 0; the caller syncs)
__device__ __forceinline__ void word_scan(const int* cnt, int* pre, int W) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int base = 0;
    for (int w0 = 0; w0 < W; w0 += 32) {
      const int v = w0 + lane < W ? cnt[w0 + lane] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (w0 + lane < W) pre[w0 + lane] = base + incl - v;
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// Dynamic shared memory: the row's scores (N floats) then the radix histogram.
template <int SW, int RQ, int SPB>
__global__ void US_SEL_LAUNCH_BOUNDS select_fused_kernel(const ProxyArgs pa, const SelectArgs sa) {
  extern __shared__ __align__(16) uint8_t fsm[];
  float* sc = reinterpret_cast<float*>(fsm);
  uint32_t* hist = reinterpret_cast<uint32_t*>(fsm + size_t(sa.N) * 4);
  float* fac_sh = reinterpret_cast<float*>(hist + kRadixBins);  // [key tiles][RQ] (c = 8 fast path)
  __shared__ float lse_sh[128];
  __shared__ double dsh[kFusedWarps];
  __shared__ int ish[kFusedWarps];
  __shared__ int wcnt[kFusedMaxW], wpre[kFusedMaxW];
  __shared__ uint32_t wbits[kFusedMaxW];
  __shared__ uint32_t ush[kFusedWarps];
  __shared__ uint32_t sh_bin, sh_above;
  __shared__ int sh_ties, sh_cert;
  __shared__ double sh_cum;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const int N = sa.N, W = sa.W;
  const long long planes = sa.rows / N;
  const int rq = RQ > 0 ? RQ : pa.rq;
  for (long long rr = blockIdx.x; rr < sa.rows; rr += gridDim.x) {
    const int plane = int(rr % planes);
    const int i = N - 1 - int(rr / planes);
    const long long row = (long long)plane * N + i;
    const int n = i + 1;
    if (tid < rq) lse_sh[tid] = pa.lse2[(long long)plane * pa.Lq + (long long)i * rq + tid];
    __syncthreads();
    constexpr bool kFac = RQ > 0 && SPB > 0;  // c = 8 fast path: per-(tile, row) factors in smem
    if (kFac) {
      proxy_tile_factors<(RQ > 0 ? RQ : 1)>(pa, plane, i, lse_sh, fac_sh, proxy_tiles_for_row(pa, i), tid,
                                           kFusedThreads);
      __syncthreads();
    }
    // ---- scores of the row (raw values to sa.scores_out when requested)
    double part = 0.0;
    bool bad = false, nonfinite = false;
    // four scores per thread in flight (their partial loads issued together);
    // indices past the row are clamped for the loads and discarded
    for (int j0 = tid; j0 < n; j0 += US_SEL_INFLIGHT * kFusedThreads) {
      float fv[US_SEL_INFLIGHT];
#pragma unroll
      for (int u = 0; u < US_SEL_INFLIGHT; ++u) {
        const int jj = min(j0 + u * kFusedThreads, n - 1);
        if constexpr (kFac) fv[u] = proxy_block_score_fac<SW, (RQ > 0 ? RQ : 1), (SPB > 0 ? SPB : 1)>(pa, plane, i, jj, fac_sh);
        else fv[u] = proxy_block_score<SW, RQ, SPB>(pa, plane, i, jj, lse_sh);
      }
#pragma unroll
      for (int u = 0; u < US_SEL_INFLIGHT; ++u) {
        const int j = j0 + u * kFusedThreads;
        if (j < n) {
          float f = fv[u];
          if (sa.scores_out) sa.scores_out[row * N + j] = f;
          if (!(f >= 0.f)) {
            bad = true;
            f = 0.f;
          }
          if (f == 0.f) f = 0.f;  // -0 -> +0
          if (isinf(f)) nonfinite = true;
          sc[j] = f;
          part += double(f);
        }
      }
    }
    // prefetch the partials of this CTA's NEXT row into L2 while this row is selected
    // (rows are read once from DRAM; the selection phases issue no loads)
    if (US_SEL_PREFETCH) {
      const long long rn = rr + gridDim.x;
      if (rn < sa.rows) {
        const int plane2 = int(rn % planes), i2 = N - 1 - int(rn / planes);
        const int nt = ((i2 + 1) * pa.rk + kProxyKeys - 1) / kProxyKeys;  // key tiles holding j <= i2
        const int ns = kProxyKeys / pa.sw;                                   // slots per key tile
        const int lines = (rq * ns * 4 + 127) / 128;                          // 128-B lines of one tile's partials
        for (int e = tid; e < nt * (lines + 1); e += kFusedThreads) {
          const int t = e / (lines + 1), u = e % (lines + 1);
          const long long base = ((long long)plane2 * pa.T + t) * pa.Lq + (long long)i2 * rq;
          const char* ptr = u < lines ? reinterpret_cast<const char*>(pa.part + base * ns) + u * 128
                                      : reinterpret_cast<const char*>(pa.tmax + base);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
        }
      }
    }
    bad = __syncthreads_or(bad);
    nonfinite = __syncthreads_or(nonfinite);
    if (bad && tid == 0) atomicOr(sa.err, 1u);
    const double total = block_sum_f64(part, dsh);

    int mode = 0;  // 0: threshold / top-k rule, 1: all, 2: diagonal only
    uint32_t bstar = 0;
    int ties_needed = 0, E_sh = 0;
    bool certified = true;
    double cum = 0.0;
    const bool topk = sa.select_mode == US_SELECT_TOP_K;
    if (!topk) {
      if (!(total > 0.0)) mode = 2;
      else if (sa.P >= 1.0) mode = 1;
      else if (nonfinite) certified = false;
    }
    if (mode == 0 && certified) {
      // ---- radix descent for v*: the largest value whose tail (mass or count)
      // reaches the target. Mass in u32 fixed point x * 2^fs with the row total
      // below 2^31 (native shared-memory integer atomics); the candidate is only
      // approximately ordered against T — certification below decides.
      const int kk = min(sa.top_k, n);
      int ex = 0;
      frexp(total > 0.0 ? total : 1.0, &ex);  // total < 2^ex
      const int fs = 30 - ex;
      const double fscale = ldexp(1.0, fs);
      const float fscale_f = ldexpf(1.0f, fs);  // x * 2^fs < 2^30: exact in fp32
      const uint32_t target = topk ? uint32_t(kk) : uint32_t(fmin(sa.P * total * fscale, 2147483647.0));
      uint32_t prefix = 0, pmask = 0, above = 0;
      // 8-bit digits: bits [30:23] (the exponent), [22:15], [14:7], [6:0]; 256 bins,
      // two per thread
#pragma unroll 1
      for (int pass = 0; pass < 4; ++pass) {
        const int sh = pass == 0 ? 23 : (pass == 1 ? 15 : (pass == 2 ? 7 : 0));
        const uint32_t dmask = pass == 3 ? 127u : 255u;
        hist[tid] = 0u;
        hist[tid + kFusedThreads] = 0u;
        __syncthreads();
#if US_SEL_AGG
        // one shared-memory atomic per distinct bin per warp (integer sums: the
        // histogram is the same in any order)
        for (int jb = tid - lane; jb < n; jb += kFusedThreads) {
          const int j = jb + lane;
          const uint32_t x = j < n ? __float_as_uint(sc[j]) : 0u;
          const bool in = j < n && (x & pmask) == prefix;
          const uint32_t bin = in ? (x >> sh) & dmask : 0xFFFFFFFFu;
          const uint32_t v = in ? (topk ? 1u : uint32_t(__uint_as_float(x) * fscale_f)) : 0u;
          const unsigned peers = __match_any_sync(0xffffffffu, bin);
          const uint32_t sum = __reduce_add_sync(peers, v);
          if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], sum);
        }
#else
        for (int j = tid; j < n; j += kFusedThreads) {
          const uint32_t x = __float_as_uint(sc[j]);
          if ((x & pmask) == prefix) atomicAdd(&hist[(x >> sh) & dmask], topk ? 1u : uint32_t(sc[j] * fscale_f));
        }
#endif
        __syncthreads();
        // exclusive suffix over threads of their two bins: warp suffix scan, then the warps above
        const uint32_t h0 = hist[2 * tid], h1 = hist[2 * tid + 1];
        const uint32_t loc = h0 + h1;
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_down_sync(0xffffffffu, incl, o);
          if (lane + o < 32) incl += y;
        }
        if (lane == 0) ush[wid] = incl;
        if (tid == 0) {
          sh_bin = 0;
          sh_above = above;
        }
        __syncthreads();
        uint32_t acc = above + (incl - loc);
#pragma unroll
        for (int w = kFusedWarps - 1; w > 0; --w)
          if (w > wid) acc += ush[w];
        // bins 2 tid + 1 (upper) then 2 tid: the crossing bin (at most one thread)
        if (acc < target && acc + h1 >= target) {
          sh_bin = uint32_t(2 * tid + 1);
          sh_above = acc;
        } else if (acc + h1 < target && acc + h1 + h0 >= target) {
          sh_bin = uint32_t(2 * tid);
          sh_above = acc + h1;
        }
        __syncthreads();
        prefix |= sh_bin << sh;
        pmask |= dmask << sh;
        above = sh_above;
      }
      bstar = prefix;
      // ---- exact fp64 boundary (+ certification for Top-P)
      double A = 0.0;
      int gt = 0, E = 0;
      for (int j = tid; j < n; j += kFusedThreads) {
        const uint32_t x = __float_as_uint(sc[j]);
        if (x > bstar) {
          A += double(sc[j]);
          ++gt;
        }
        if (x == bstar) ++E;
      }
      A = block_sum_f64(A, dsh);
      gt = block_sum_i32(gt, ish);
      E = block_sum_i32(E, ish);
      E_sh = E;
      if (topk) {
        ties_needed = kk - gt;
      } else {
        if (tid == 0) {
          const double T = sa.P * total;
          const double eps = 4.0 * double(n) * 0x1p-53 * total;
          const double vstar = double(__uint_as_float(bstar));
          double c = A;
          bool cert = (T - c) > eps;
          int k = 0;
          while (k < E) {
            c += vstar;
            ++k;
            if (c >= T) break;
            cert = cert && (T - c) > eps;
          }
          cert = cert && (c >= T) && (c - T) > eps;
          sh_ties = k;
          sh_cum = c;
          sh_cert = cert ? 1 : 0;
        }
        __syncthreads();
        ties_needed = sh_ties;
        cum = sh_cum;
        certified = sh_cert != 0;
      }
    }
    if (!certified) {
      // exact sorted walk (select_fallback_fused_kernel recomputes the row)
      if (tid == 0) sa.fb_rows[atomicAdd(sa.fb_count, 1)] = int32_t(row);
      __syncthreads();
      continue;
    }
    // ---- emit: bits, counts, coverage, ascending indices. Ties of v* need ranks
    // (ascending index) only when some but not all of them are taken.
    const int nw = (n + 31) >> 5;  // words that can hold selected bits
    const bool tie_ranks = mode == 0 && ties_needed > 0 && ties_needed < E_sh;
    if (tie_ranks) {
      for (int w = wid; w < nw; w += kFusedWarps) {
        const int idx = w * 32 + lane;
        const bool tie = idx < n && __float_as_uint(sc[idx]) == bstar;
        const uint32_t tm = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wcnt[w] = __popc(tm);
      }
      __syncthreads();
      word_scan(wcnt, wpre, nw);
      __syncthreads();
    }
    double smass = 0.0;
    int cnt = 0;
    for (int w = wid; w < W; w += kFusedWarps) {
      const int idx = w * 32 + lane;
      const bool valid = idx < n;
      bool sel;
      if (mode == 1) {
        sel = valid;
      } else if (mode == 2) {
        sel = idx == n - 1;
      } else {
        const uint32_t x = valid ? __float_as_uint(sc[idx]) : 0u;
        const bool tie = valid && x == bstar;
        if (tie_ranks) {
          const uint32_t tm = __ballot_sync(0xffffffffu, tie);
          sel = valid && (x > bstar || (tie && wpre[w] + __popc(tm & lt_mask) < ties_needed));
        } else {
          sel = valid && (x > bstar || (tie && ties_needed > 0));
        }
      }
      const uint32_t word = __ballot_sync(0xffffffffu, sel);
      if (sel && topk) smass += double(sc[idx]);
      cnt += __popc(word);
      if (lane == 0) {
        sa.mask_bits[row * W + w] = word;
        if (w < nw) wbits[w] = word;
      }
    }
    const int count = block_sum_i32(lane == 0 ? cnt : 0, ish);
    if (sa.indices) {
      if (tid < nw) wcnt[tid] = __popc(wbits[tid]);
      __syncthreads();
      word_scan(wcnt, wpre, nw);
      __syncthreads();
      for (int w = wid; w < nw; w += kFusedWarps) {
        const uint32_t word = wbits[w];
        if ((word >> lane) & 1u) sa.indices[row * N + wpre[w] + __popc(word & lt_mask)] = int16_t(w * 32 + lane);
      }
    }
    const double m = topk ? block_sum_f64(smass, dsh) : 0.0;
    if (tid == 0) {
      double cov;
      if (topk) cov = total > 0.0 ? m / total : 1.0;
      else cov = mode == 0 ? cum / total : 1.0;
      if (sa.counts) sa.counts[row] = count;
      if (sa.coverage) sa.coverage[row] = cov;
    }
    __syncthreads();
  }
}

// Exact reference walk for the fused path's uncertified rows: the row's scores are
// recomputed from the partials (same arithmetic), then the sorted fp64 walk of
// select_fallback_kernel.
template <int SW, int RQ, int SPB>
__global__ void __launch_bounds__(256) select_fallback_fused_kernel(const ProxyArgs pa, SelectArgs a) {
  __shared__ unsigned long long keys[kFbMaxN];
  __shared__ uint8_t flag[kFbMaxN];
  __shared__ float lse_sh[128];
  __shared__ float fac_fb[kMaxFacTiles * 8];
  __shared__ int sh_k;
  __shared__ double sh_cov;
  const int count = *a.fb_count;
  const int rq = RQ > 0 ? RQ : pa.rq;
  for (int e = blockIdx.x; e < count; e += gridDim.x) {
    const long long row = a.fb_rows[e];
    const int plane = int(row / a.N), i = int(row % a.N), n = i + 1;
    if (threadIdx.x < rq) lse_sh[threadIdx.x] = pa.lse2[(long long)plane * pa.Lq + (long long)i * rq + threadIdx.x];
    __syncthreads();
    constexpr bool kFac = RQ > 0 && SPB > 0;
    if (kFac) {
      proxy_tile_factors<(RQ > 0 ? RQ : 1)>(pa, plane, i, lse_sh, fac_fb, proxy_tiles_for_row(pa, i), threadIdx.x,
                                           blockDim.x);
      __syncthreads();
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int t = threadIdx.x; t < n2; t += blockDim.x) {
      if (t < n) {
        float f;
        if constexpr (kFac) f = proxy_block_score_fac<SW, (RQ > 0 ? RQ : 1), (SPB > 0 ? SPB : 1)>(pa, plane, i, t, fac_fb);
        else f = proxy_block_score<SW, RQ, SPB>(pa, plane, i, t, lse_sh);
        if (!(f >= 0.f) || f == 0.f) f = 0.f;
        keys[t] = ((unsigned long long)(~__float_as_uint(f)) << 32) | unsigned(t);
      } else {
        keys[t] = ~0ull;
      }
      flag[t] = 0;
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = threadIdx.x; t < n2; t += blockDim.x) {
          const int p = t ^ j;
          if (p > t) {
            const unsigned long long x = keys[t], y = keys[p];
            const bool up = (t & k) == 0;
            if ((x > y) == up) {
              keys[t] = y;
              keys[p] = x;
            }
          }
        }
        __syncthreads();
      }
    if (threadIdx.x == 0) {
      auto val = [&](int t) { return double(__uint_as_float(~unsigned(keys[t] >> 32))); };
      double total = 0.0;
      for (int t = 0; t < n; ++t) total += val(t);
      int ksel;
      double cov = 1.0;
      if (total <= 0.0) {
        ksel = -1;
      } else if (a.P >= 1.0) {
        ksel = n;
      } else {
        double cum = 0.0;
        ksel = 0;
        for (int t = 0; t < n; ++t) {
          ++ksel;
          cum += val(t);
          if (cum >= a.P * total) break;
        }
        cov = cum / total;
      }
      sh_k = ksel;
      sh_cov = cov;
    }
    __syncthreads();
    const int ksel = sh_k;
    if (ksel < 0) {
      if (threadIdx.x == 0) flag[n - 1] = 1;
    } else {
      for (int t = threadIdx.x; t < ksel; t += blockDim.x) flag[unsigned(keys[t] & 0xFFFFFFFFu)] = 1;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int base = 0;
      for (int w = 0; w < a.W; ++w) {
        const int idx = w * 32 + lane;
        const bool sel = idx < n && flag[idx];
        const uint32_t word = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) a.mask_bits[row * a.W + w] = word;
        if (a.indices && sel) a.indices[row * a.N + base + __popc(word & ((1u << lane) - 1u))] = int16_t(idx);
        base += __popc(word);
      }
      if (lane == 0) {
        if (a.counts) a.counts[row] = base;
        if (a.coverage) a.coverage[row] = sh_cov;
      }
    }
    __syncthreads();
  }
}

template <int SW, int RQ, int SPB>
void launch_fused_t(const ProxyArgs& pa, const SelectArgs& sa, cudaStream_t st) {
  // scores + bins + the per-(tile, row) factors of the c = 8 path: <= 25 KB (no attribute needed)
  const int smem = sa.N * 4 + kRadixBins * 4 + (RQ > 0 && SPB > 0 ? kMaxFacTiles * RQ * 4 : 0);
  long long blocks = sa.rows;
  if (blocks > 148 * US_SEL_GRID_PER_SM) blocks = 148 * US_SEL_GRID_PER_SM;
  select_fused_kernel<SW, RQ, SPB><<<unsigned(blocks), kFusedThreads, smem, st>>>(pa, sa);
  if (sa.select_mode == US_SELECT_TOP_P) select_fallback_fused_kernel<SW, RQ, SPB><<<148, 256, 0, st>>>(pa, sa);
}

__global__ void mask_check_kernel(const uint32_t* mask, int rows, int N, int W, uint32_t* err,
                                  int32_t* first_bad) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int i = int(row % N);
  const uint32_t* m = mask + row * W;
  bool any = false, noncausal = false;
  for (int w = 0; w < W; ++w) {
    uint32_t word = m[w];
    const int lo = w * 32;
    uint32_t causal_bits;
    if (lo + 31 <= i) causal_bits = ~0u;
    else if (lo > i) causal_bits = 0u;
    else causal_bits = (i - lo == 31) ? ~0u : ((1u << (i - lo + 1)) - 1u);
    if (word & ~causal_bits) noncausal = true;
    if (word & causal_bits) any = true;
  }
  if (noncausal) {
    atomicOr(err, 4u);
    atomicMin(first_bad, int32_t(row));
  }
  if (!any) {
    atomicOr(err, 8u);
    atomicMin(first_bad, int32_t(row));
  }
}

// S = 64 m block masks -> the 64-granular masks the attention kernels walk: query
// sub-block ii = i m + a keeps key sub-block jj = j m + b iff block (i, j) is selected,
// except the sub-blocks of the diagonal block that lie wholly in the future (j == i,
// b > a) — token-level causality inside the diagonal block is then exactly the
// 64-granular kernel's (attention.cpp:117-118). Non-causal source bits (j > i) are
// kept, so the kernels' mask checks still see them.
__global__ void mask_expand_kernel(const uint32_t* __restrict__ in, long long rows64, int N, int W, int m,
                                   int N64, int W64, uint32_t* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows64 * W64) return;
  const int w64 = int(t % W64);
  const long long r64 = t / W64;
  const int ii = int(r64 % N64);
  const long long plane = r64 / N64;
  const int i = ii / m;
  const uint32_t* src = in + (plane * N + i) * W;
  uint32_t word = 0;
#pragma unroll 4
  for (int b = 0; b < 32; ++b) {
    const int jj = w64 * 32 + b;
    if (jj >= N64) break;
    const int j = jj / m;
    const bool sel = (src[j >> 5] >> (j & 31)) & 1u;
    if (sel && !(j == i && jj > ii)) word |= 1u << b;
  }
  out[t] = word;
}

template <int NPL>
void launch_sel(const SelectArgs& a, cudaStream_t st) {
  const int threads = 256, wpc = threads / 32;
  long long blocks = (a.rows + wpc - 1) / wpc;
  if (blocks > 148 * 16) blocks = 148 * 16;
  select_kernel<NPL><<<unsigned(blocks), threads, 0, st>>>(a);
}

}  // namespace

us_status launch_select(const SelectArgs& a, cudaStream_t st) {
  if (a.N > kFbMaxN) {
    set_error("select: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  const int npl = (a.N + 31) / 32;
  if (npl <= 1) launch_sel<1>(a, st);
  else if (npl <= 2) launch_sel<2>(a, st);
  else if (npl <= 4) launch_sel<4>(a, st);
  else if (npl <= 8) launch_sel<8>(a, st);
  else if (npl <= 16) launch_sel<16>(a, st);
  else if (npl <= 32) launch_sel<32>(a, st);
  else if (npl <= 64) launch_sel<64>(a, st);
  else launch_sel<128>(a, st);
  US_LAUNCH_CHECK("select_kernel");
  if (a.select_mode == US_SELECT_TOP_P) {
    select_fallback_kernel<<<148, 256, 0, st>>>(a);
    US_LAUNCH_CHECK("select_fallback_kernel");
  }
  return US_OK;
}

us_status launch_select_fused(const ProxyArgs& pa, const SelectArgs& sa, cudaStream_t st) {
  if (sa.N > kFbMaxN) {
    set_error("select: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (pa.sw == 8 && pa.rq == 8 && pa.rk == 8) launch_fused_t<8, 8, 1>(pa, sa, st);
  else if (pa.sw == 8) launch_fused_t<8, 0, 0>(pa, sa, st);
  else if (pa.sw == 4) launch_fused_t<4, 0, 0>(pa, sa, st);
  else if (pa.sw == 2) launch_fused_t<2, 0, 0>(pa, sa, st);
  else launch_fused_t<1, 0, 0>(pa, sa, st);
  US_LAUNCH_CHECK("select_fused_kernel");
  if (sa.select_mode == US_SELECT_TOP_P) US_LAUNCH_CHECK("select_fallback_fused_kernel");
  return US_OK;
}

us_status launch_mask_expand(const uint32_t* in, long long planes, int N, int W, int m, uint32_t* out,
                             cudaStream_t st) {
  const int N64 = N * m, W64 = (N64 + 31) / 32;
  const long long n = planes * N64 * W64;
  mask_expand_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(in, planes * N64, N, W, m, N64, W64, out);
  US_LAUNCH_CHECK("mask_expand_kernel");
  return US_OK;
}

us_status launch_mask_check(const uint32_t* mask, int rows, int N, int W, uint32_t* err,
                            int32_t* first_bad, cudaStream_t st) {
  mask_check_kernel<<<(rows + 255) / 256, 256, 0, st>>>(mask, rows, N, W, err, first_bad);
  US_LAUNCH_CHECK("mask_check_kernel");
  return US_OK;
}

}  // namespace us
