// proxy_score.cuh — the block score of one (query block i, key block j <= i) from
// the proxy kernel's slot partials (block_aggregate, proxy.cpp:48-72):
//     score(i, j) = sum_{rows r of block i} 2^(m_t(r) - lse2(r)) * sum_{slots of j} P_t(r)[s]
// in a fixed order (rows r = 0..rq-1, slots ascending). Shared by the standalone
// finalize (proxy.cu) and the fused finalize + selection kernel (select.cu), so both
// produce bit-identical f32 scores.
#pragma once
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {

constexpr int kProxyKeys = 128;  // composite keys per proxy key tile (UMMA N)

// RQ / SPB > 0: compile-time rows per query block / slots per key block (the c = 8
// fast path: every load of a score issued before its first use). lse_sh holds the
// rq row LSEs of query block i (log2 units).
template <int SW, int RQ, int SPB>
__device__ __forceinline__ float proxy_block_score(const ProxyArgs& a, int plane, int i, int j,
                                                   const float* lse_sh) {
  constexpr int NS = kProxyKeys / SW;
  const int rq = RQ > 0 ? RQ : a.rq;
  const int spb = SPB > 0 ? SPB : a.rk / SW;  // slots per key block
  const int row0 = i * rq;
  const int key0 = j * a.rk;
  const int t = key0 / kProxyKeys, s0 = (key0 % kProxyKeys) / SW;
  const long long base = ((long long)plane * a.T + t) * a.Lq + row0;
  float acc = 0.f;
  if (RQ > 0 && SPB > 0) {
    constexpr int R = RQ > 0 ? RQ : 1;
    float pm[R], ps[R];
#pragma unroll
    for (int r = 0; r < RQ; ++r) {
      pm[r] = __ldg(a.tmax + base + r);
      float v = 0.f;
#pragma unroll
      for (int u = 0; u < SPB; ++u) v += __ldg(a.part + (base + r) * NS + s0 + u);
      ps[r] = v;
    }
    // (a row with no live key — a competitor proxy's first phase-class row — adds 0)
#pragma unroll
    for (int r = 0; r < RQ; ++r) acc += lse_sh[r] == -INFINITY ? 0.f : ps[r] * ex2_approx(pm[r] - lse_sh[r]);
  } else {
    for (int r = 0; r < rq; ++r) {
      const float* pr = a.part + (base + r) * NS + s0;
      float v = 0.f;
      for (int u = 0; u < spb; ++u) v += pr[u];
      acc += lse_sh[r] == -INFINITY ? 0.f : v * ex2_approx(a.tmax[base + r] - lse_sh[r]);
    }
  }
  return acc;
}

// The c = 8 fast path with per-(key tile, row) factors precomputed once per query
// block: fac[t * RQ + r] = 2^(m_t(r) - lse2(r)) (0 for a row with no live key), so a
// score costs RQ partial loads and RQ multiply-adds instead of RQ tile-max loads and
// exponentials more. Explicit _rn operations (no contraction): every kernel that
// evaluates a score gets the identical f32 value.
template <int RQ>
__device__ __forceinline__ void proxy_tile_factors(const ProxyArgs& a, int plane, int i, const float* lse_sh,
                                                   float* fac, int n_tiles, int tid, int nthreads) {
  for (int e = tid; e < n_tiles * RQ; e += nthreads) {
    const int t = e / RQ, r = e % RQ;
    const float l = lse_sh[r];
    fac[e] = l == -INFINITY ? 0.f
                            : ex2_approx(__ldg(a.tmax + ((long long)plane * a.T + t) * a.Lq + (long long)i * RQ + r) - l);
  }
}
template <int SW, int RQ, int SPB>
__device__ __forceinline__ float proxy_block_score_fac(const ProxyArgs& a, int plane, int i, int j, const float* fac) {
  constexpr int NS = kProxyKeys / SW;
  const int key0 = j * a.rk;
  const int t = key0 / kProxyKeys, s0 = (key0 % kProxyKeys) / SW;
  const long long base = ((long long)plane * a.T + t) * a.Lq + (long long)i * RQ;
  float ps[RQ];
#pragma unroll
  for (int r = 0; r < RQ; ++r) {
    float v = 0.f;
#pragma unroll
    for (int u = 0; u < SPB; ++u) v = __fadd_rn(v, __ldg(a.part + (base + r) * NS + s0 + u));
    ps[r] = v;
  }
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r < RQ; ++r) acc = __fadd_rn(acc, __fmul_rn(ps[r], fac[t * RQ + r]));
  return acc;
}
// key tiles holding the key blocks j <= i of query block i
__device__ __forceinline__ int proxy_tiles_for_row(const ProxyArgs& a, int i) {
  return ((i + 1) * a.rk + kProxyKeys - 1) / kProxyKeys;
}

}  // namespace us
