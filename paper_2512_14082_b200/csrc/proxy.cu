// proxy.cu — compressed proxy attention on tcgen05.
//
// Reference: compressed_attention (proxy.cpp:10-46) and block_aggregate
// (proxy.cpp:48-72): logits = Qc.Kc^T / sqrt(d) in fp64, softmax per composite
// row over all composite keys (post-softmax, the default) or over the live
// prefix (pre-softmax, live iff (t'+1)c_q - 1 >= s' c_k), then per
// (query block i, key block j <= i) region sums.
//
// Precision ("fp16x3"): Qc/Kc are f32. The split kernel stores x * 2^e as
// hi = fp16(x 2^e), lo = fp16(x 2^e - hi) (~22 significant bits). Each logit
// tile is accumulated by three tcgen05 MMAs into one fp32 TMEM accumulator:
// hi.hi + hi.lo + lo.hi (the dropped lo.lo term is < 2^-22 relative). This is
// fp32-class accuracy at f16 tensor-core rate — plain bf16/tf32 composite
// tokens flip mask bits vs the fp64 reference.
//
// ONE pass over the logits. Post-softmax needs each row's LSE over every key
// before any probability is known, so instead of recomputing the causal half
// (a second MMA pass), each row keeps, per causal key tile t, the tile max
// m_t and the slot sums P_t[s] = sum_{keys in slot s} 2^(x - m_t) (a slot is
// SW = min(rk, 8) consecutive composite keys, so every key block is a whole
// number of slots), written to HBM; the row LSE accumulates online. The
// finalize kernel then forms
//     score(i, j) = sum_{rows r of block i} 2^(m_t(r) - lse2(r)) * sum_{slots of j} P_t(r)[s]
// in a fixed order. Cost: 1x the full-square MMA work (was 1.5x) plus
// Lq * N * 4 bytes of slot partials per plane written and read once.
//
// CTA = 128 composite query rows (UMMA M = 128) of one compressed head; key
// tiles of 128 composite keys (N = 128). Q hi/lo live in TMEM (TS-mode MMAs:
// the A operand is read from TMEM, which measured 71.5 vs 96.3 cycles per
// M=128/N=128/K=16 MMA against SMEM A, profiles/r01_summary.md); only K tiles
// are streamed through SMEM by TMA.
// Roles (320 threads): warp 0 TMA producer (K ring), warp 1 MMA issuer + TMEM
// owner, warps 2-5 epilogue group 0 (even tiles, S buffer 0), warps 6-9
// epilogue group 1 (odd tiles, S buffer 1). Epilogue warp w owns TMEM lanes
// 32 * (w % 4) (thread = composite row); the two groups keep independent
// online (max, sum) per row and merge them at the end.
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"
#include "proxy_score.cuh"

namespace us {
namespace {

constexpr int kRows = 128;  // composite query rows per CTA (UMMA M)
constexpr int kKeys = kProxyKeys;  // composite keys per tile (UMMA N)
// TMEM columns: S buffers [0,128) and [128,256); Q hi at 256, Q lo at 320 (D/2 cols each).
constexpr uint32_t kTS0 = 0, kTQh = 256, kTQl = 320;
// K-tile producer warps: one TMA-issuing warp sustains only ~20-29 B/clk of copies
// (profiles/r02d/tma_probe.txt) while the fp16x3 MMAs consume a 64 KB hi+lo tile per
// ~1700-2000 cycles (33-38 B/clk); with 2, warp 10 issues the second d-chunk of every tile.
#ifndef US_PROXY_FMA  // 1: exponent arguments as one FFMA2 of the raw logits (see the epilogue)
#define US_PROXY_FMA 1
#endif
#ifndef US_PROXY_FADD2  // 1: the slot sums' additions paired into FADD2 (same operands, same order)
#define US_PROXY_FADD2 0
#endif
#ifndef US_PROXY_FULLTILE  // 1: tiles whose keys are all live skip the per-key live test
#define US_PROXY_FULLTILE 1
#endif
#ifndef US_PROXY_KPROD
#define US_PROXY_KPROD 1
#endif
constexpr int kKProd = US_PROXY_KPROD;
constexpr int kProxyThreads = (10 + (kKProd - 1)) * 32;

template <int D>
struct ProxySmem {
  static constexpr int kChunks = D / 64;          // 128-byte swizzle atoms along d
  static constexpr int kKBytes = kKeys * D * 2;   // one of hi / lo
  static constexpr int kStages = D == 128 ? 3 : 6;
  static constexpr int kBytes = kStages * 2 * kKBytes;
};

__device__ __forceinline__ int live_keys(int t, int c_q, int c_k, int Lk, int mode) {
  if (mode == US_POST_SOFTMAX_BLOCK_CAUSAL) return Lk;
  const long long last_q = (long long)(t + 1) * c_q - 1;
  const long long live = last_q / c_k + 1;
  return live < Lk ? int(live) : Lk;
}

template <int D, int SW, bool X3>
__global__ void __launch_bounds__(kProxyThreads, 1)
    proxy_kernel(const __grid_constant__ CUtensorMap tmKh, const __grid_constant__ CUtensorMap tmKl,
                 const ProxyArgs a) {
  using L = ProxySmem<D>;
  constexpr int kST = L::kStages;
  constexpr int NS = kKeys / SW;  // slots per key tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_kfull[kST], bar_kempty[kST], bar_sfull[2], bar_sempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float2 ml_sh[kRows];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rt = gridDim.x - 1 - blockIdx.x;
  const int hc = blockIdx.y, b = blockIdx.z;
  const int r0 = rt * kRows;
  const int plane = b * a.Hc + hc;
  const int kplane = b * a.kv_planes + (hc * a.kv_mul) / a.kv_div;

  const int r_last = min(r0 + kRows, a.Lq) - 1;
  // X3: UniSparse composite rows (live rule of the causal mode); !X3: strided raw rows
  // of a competitor proxy, live keys = row + live_bias (causal by original position)
  const int nkeys = X3 ? live_keys(r_last, a.c_q, a.c_k, a.Lk, a.causal_mode) : min(a.Lk, r_last + a.live_bias);
  const int n_tiles = (nkeys + kKeys - 1) / kKeys;
  const int i_max = r_last / a.rq;
  const int causal_keys = min(a.Lk, (i_max + 1) * a.rk);
  const int n_part_tiles = X3 ? min(n_tiles, (causal_keys + kKeys - 1) / kKeys) : n_tiles;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 8);
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kfull[s], X3 && D == 128 ? kKProd : 1);
      mbar_init(&bar_kempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sempty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0 || warp >= 10) {
    // ------------------------------------------------------------ TMA producer(s)
    // (kKProd = 2 with X3 and D = 128: warp 0 loads d-chunk 0 of hi and lo, warp 10 chunk 1)
    const int pi = warp == 0 ? 0 : 1;
    const int np = X3 && D == 128 ? kKProd : 1;
    if (pi < np && elect_one()) {
      tma_prefetch_desc(&tmKh);
      tma_prefetch_desc(&tmKl);
      const uint64_t pol = policy_evict_last();  // K tiles are re-read by every row tile
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % kST;
        if (t >= kST) mbar_wait(&bar_kempty[s], ((t / kST) + 1) & 1);
        uint8_t* kh = smem + s * 2 * L::kKBytes;
        uint8_t* kl = kh + L::kKBytes;
        const int krow = kplane * a.Lk + t * kKeys;
        if (X3) {
          mbar_arrive_expect_tx(&bar_kfull[s], 2 * L::kKBytes / np);
          for (int kc = pi; kc < L::kChunks; kc += np) {
            tma_load_2d_hint(kh + kc * kKeys * 128, &tmKh, &bar_kfull[s], kc * 64, krow, pol);
            tma_load_2d_hint(kl + kc * kKeys * 128, &tmKl, &bar_kfull[s], kc * 64, krow, pol);
          }
        } else {
          // raw bf16 K rows of one phase class: 3-D map (d, stride, rows / stride)
          mbar_arrive_expect_tx(&bar_kfull[s], L::kKBytes);
          for (int kc = 0; kc < L::kChunks; ++kc)
            tma_load_3d_hint(kh + kc * kKeys * 128, &tmKh, &bar_kfull[s], kc * 64, a.k_phase, krow, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_f16(kRows, kKeys, /*f16 or bf16*/ X3 ? 0 : 1, false, false);
    mbar_wait(&bar_q, 0);
    tc_fence_after();
    for (int t = 0; t < n_tiles; ++t) {
      const int s = t % kST, buf = t & 1;
      mbar_wait(&bar_kfull[s], (t / kST) & 1);
      if (t >= 2) mbar_wait(&bar_sempty[buf], ((t - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t kh = smem_u32(smem + s * 2 * L::kKBytes), kl = kh + L::kKBytes;
        const uint32_t d_tmem = tmem + kTS0 + buf * kKeys;
#pragma unroll
        for (int kc = 0; kc < L::kChunks; ++kc) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t ko = kc * kKeys * 128 + ks * 32;
            const uint32_t qcol = (kc * 4 + ks) * 8;
            const uint64_t bkh = sdesc_sw128(kh + ko, 16, 1024), bkl = sdesc_sw128(kl + ko, 16, 1024);
            if (X3) {
              umma_f16_ts(d_tmem, tmem + kTQh + qcol, bkl, idesc, (kc | ks) != 0);
              umma_f16_ts(d_tmem, tmem + kTQl + qcol, bkh, idesc, 1);
              umma_f16_ts(d_tmem, tmem + kTQh + qcol, bkh, idesc, 1);
            } else {
              // bf16 inputs: products are exact in fp32, one MMA per K step
              umma_f16_ts(d_tmem, tmem + kTQh + qcol, bkh, idesc, (kc | ks) != 0);
            }
          }
        }
        umma_commit(&bar_kempty[s]);
        umma_commit(&bar_sfull[buf]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue groups
    const int grp = (warp - 2) >> 2;  // 0: even tiles, 1: odd tiles
    const int q = warp & 3;           // TMEM lane quarter
    const int row = q * 32 + lane;
    const int t_row = r0 + row;
    const bool row_ok = t_row < a.Lq;
    const uint32_t lane_addr = tmem + (uint32_t(q * 32) << 16);
    {
      // Q hi (group 0) / Q lo (group 1) row -> TMEM, the A operand of every MMA
      // (!X3: group 0 stores the raw bf16 query row t = q_row0 + row * q_stride + q_phase)
      const uint16_t* src = X3 ? reinterpret_cast<const uint16_t*>((grp == 0 ? a.qh : a.ql) +
                                                                 ((long long)plane * a.Lq + t_row) * D)
                               : a.qraw + ((long long)plane * a.L + a.q_row0 + (long long)t_row * a.q_stride +
                                           a.q_phase) * D;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
      for (int c0 = 0; c0 < D / 2; c0 += 16) {
        if (!X3 && grp == 1) break;
        uint32_t w16[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 v = row_ok ? __ldg(s4 + c0 / 4 + u) : make_uint4(0, 0, 0, 0);
          w16[4 * u] = v.x;
          w16[4 * u + 1] = v.y;
          w16[4 * u + 2] = v.z;
          w16[4 * u + 3] = v.w;
        }
        tmem_st16(lane_addr + (grp == 0 ? kTQh : kTQl) + c0, w16);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_q);
    }
    const int live = !row_ok ? 0
                     : X3    ? live_keys(t_row, a.c_q, a.c_k, a.Lk, a.causal_mode)
                             : max(0, min(a.Lk, t_row + a.live_bias));
    const int eq = !X3 ? 0 : (a.q_row_exp ? (row_ok ? a.exp_q[(long long)plane * a.Lq + t_row] : 0) : a.exp_q[plane]);
    const float k2 = X3 ? ldexpf(a.scale_log2, -(eq + a.exp_k[kplane])) : a.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int t = grp; t < n_tiles; t += 2) {
      mbar_wait(&bar_sfull[grp], (t >> 1) & 1);
      tc_fence_after();
      uint32_t v[kKeys];
      {
        uint32_t* v0 = v;
        tmem_ld32(lane_addr + kTS0 + grp * kKeys + 0, *reinterpret_cast<uint32_t(*)[32]>(v0));
        tmem_ld32(lane_addr + kTS0 + grp * kKeys + 32, *reinterpret_cast<uint32_t(*)[32]>(v0 + 32));
        tmem_ld32(lane_addr + kTS0 + grp * kKeys + 64, *reinterpret_cast<uint32_t(*)[32]>(v0 + 64));
        tmem_ld32(lane_addr + kTS0 + grp * kKeys + 96, *reinterpret_cast<uint32_t(*)[32]>(v0 + 96));
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sempty[grp]);

#ifdef US_PROXY_SKELETON
      // calibration: MMA-pipeline rate with a math-free epilogue (results are garbage)
      if (v[0] == 0x7fffffffu && v[127] == 0x7fffffffu) a.tmax[0] = 1.f;
      continue;
#endif
      const int nvalid = min(max(live - t * kKeys, 0), kKeys);
      float x[kKeys];
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = -INFINITY;
#if US_PROXY_FMA
      // max over the raw logits, scaled once (k2 > 0: RN scaling is monotonic, so this is
      // the max of the scaled logits bit for bit); the exponent argument below is then one
      // FFMA2 (x k2 - mt, a single rounding) instead of a multiply and an add
#if US_PROXY_FULLTILE
      if (nvalid >= kKeys) {  // every key of the tile live (all but the last tile of a row)
#pragma unroll
        for (int c = 0; c < kKeys; ++c) {
          x[c] = __uint_as_float(v[c]);
          m8[c & 7] = fmaxf(m8[c & 7], x[c]);
        }
      } else
#endif
      {
#pragma unroll
        for (int c = 0; c < kKeys; ++c) {
          x[c] = c < nvalid ? __uint_as_float(v[c]) : -INFINITY;
          m8[c & 7] = fmaxf(m8[c & 7], x[c]);
        }
      }
      const float mraw = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      const float mt = mraw == -INFINITY ? -INFINITY : mraw * k2;
#else
#pragma unroll
      for (int c = 0; c < kKeys; ++c) {
        x[c] = c < nvalid ? __uint_as_float(v[c]) * k2 : -INFINITY;
        m8[c & 7] = fmaxf(m8[c & 7], x[c]);
      }
      const float mt = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                             fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
#endif
      // slot sums (fixed pairwise order inside each slot of SW keys)
      float slot[NS];
      if (mt == -INFINITY) {
#pragma unroll
        for (int s = 0; s < NS; ++s) slot[s] = 0.f;
      } else {
        const float2 nm = make_float2(-mt, -mt);
#if US_PROXY_FMA
        const float2 kk = make_float2(k2, k2);
#endif
#pragma unroll
        for (int c = 0; c < kKeys; c += 2) {
#if US_PROXY_FMA
          const float2 d2 = __ffma2_rn(make_float2(x[c], x[c + 1]), kk, nm);
#else
          const float2 d2 = __fadd2_rn(make_float2(x[c], x[c + 1]), nm);
#endif
          x[c] = ex2_approx(d2.x);
          x[c + 1] = ex2_approx(d2.y);
        }
#if US_PROXY_FADD2
        // the same additions, two per FADD2 (x[c] += x[c + w] and x[c + 2w] += x[c + 3w])
#pragma unroll
        for (int w = 1; w < SW; w <<= 1)
#pragma unroll
          for (int c = 0; c < kKeys; c += 4 * w) {
            const float2 r = __fadd2_rn(make_float2(x[c], x[c + 2 * w]), make_float2(x[c + w], x[c + 3 * w]));
            x[c] = r.x;
            x[c + 2 * w] = r.y;
          }
#else
#pragma unroll
        for (int w = 1; w < SW; w <<= 1)
#pragma unroll
          for (int c = 0; c < kKeys; c += 2 * w) x[c] += x[c + w];
#endif
#pragma unroll
        for (int s = 0; s < NS; ++s) slot[s] = x[s * SW];
      }
      float tot = 0.f;
      {
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < NS; ++s) acc4[s & 3] += slot[s];
        tot = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      }
      if (mt > m) {
        l = l * ex2_approx(m - mt) + tot;
        m = mt;
      } else if (mt != -INFINITY) {
        l += tot * ex2_approx(mt - m);
      }
      if (t < n_part_tiles && row_ok) {
        const long long prow = ((long long)plane * a.T + t) * a.Lq + t_row;
        float4* dst = reinterpret_cast<float4*>(a.part + prow * NS);
#pragma unroll
        for (int s = 0; s < NS; s += 4) dst[s / 4] = make_float4(slot[s], slot[s + 1], slot[s + 2], slot[s + 3]);
        a.tmax[prow] = mt;
      }
    }
    // merge the two groups' online (max, sum) per row -> row LSE in log2 units
    if (grp == 1) ml_sh[row] = make_float2(m, l);
    named_bar_sync(1, 256);
    if (grp == 0 && row_ok) {
      const float2 o = ml_sh[row];
      const float M = fmaxf(m, o.x);
      const float lt = (m == -INFINITY ? 0.f : l * ex2_approx(m - M)) + (o.x == -INFINITY ? 0.f : o.y * ex2_approx(o.x - M));
      a.lse2[(long long)plane * a.Lq + t_row] = M + __log2f(lt);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// score(i, j) for j <= i from the slot partials (proxy_score.cuh). CTA = (query
// block i, plane). Only used when the scores tensor itself is wanted (competitor
// proxies, exact block mass); the UniSparse path fuses this into the selection
// (select.cu, launch_select_fused).
template <int SW, int RQ, int SPB>
__global__ void __launch_bounds__(256) proxy_finalize_kernel(const ProxyArgs a) {
  __shared__ float lse_sh[128];
  const int i = gridDim.x - 1 - blockIdx.x;
  const int plane = blockIdx.y;
  const int rq = RQ > 0 ? RQ : a.rq;
  if (threadIdx.x < rq) lse_sh[threadIdx.x] = a.lse2[(long long)plane * a.Lq + i * rq + threadIdx.x];
  __syncthreads();
  constexpr bool kFac = RQ > 0 && SPB > 0;
  __shared__ float fac[kFac ? 256 * (RQ > 0 ? RQ : 1) : 1];
  if (kFac) {
    proxy_tile_factors<(RQ > 0 ? RQ : 1)>(a, plane, i, lse_sh, fac, proxy_tiles_for_row(a, i), threadIdx.x, blockDim.x);
    __syncthreads();
  }
  float* out = a.scores + ((long long)plane * a.N + i) * a.N;
  for (int j = threadIdx.x; j <= i; j += blockDim.x) {
    float acc;
    if constexpr (kFac) acc = proxy_block_score_fac<SW, (RQ > 0 ? RQ : 1), (SPB > 0 ? SPB : 1)>(a, plane, i, j, fac);
    else acc = proxy_block_score<SW, RQ, SPB>(a, plane, i, j, lse_sh);
    out[j] = a.accumulate ? out[j] + acc : acc;
  }
}

template <int D, int SW, bool X3>
us_status launch_proxy_x(const ProxyArgs& a, const CUtensorMap& tmKh, const CUtensorMap& tmKl, cudaStream_t st) {
  const int smem = ProxySmem<D>::kBytes + 1024;
  auto kern = proxy_kernel<D, SW, X3>;
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(kern, smem, attr_done, "proxy_kernel smem attribute"); s != US_OK) return s;
  dim3 grid((a.Lq + kRows - 1) / kRows, a.Hc, a.B);
  kern<<<grid, kProxyThreads, smem, st>>>(tmKh, tmKl, a);
  US_LAUNCH_CHECK("proxy_kernel");
  if (!a.finalize) return US_OK;
  const dim3 fgrid(a.N, a.B * a.Hc);
  if (SW == 8 && a.rq == 8 && a.rk == 8) proxy_finalize_kernel<SW, 8, 1><<<fgrid, 256, 0, st>>>(a);
  else proxy_finalize_kernel<SW, 0, 0><<<fgrid, 256, 0, st>>>(a);
  US_LAUNCH_CHECK("proxy_finalize_kernel");
  return US_OK;
}

template <int D, int SW>
us_status launch_proxy_t(const ProxyArgs& a, const CUtensorMap& tmKh, const CUtensorMap& tmKl, cudaStream_t st) {
  return a.x3 ? launch_proxy_x<D, SW, true>(a, tmKh, tmKl, st) : launch_proxy_x<D, SW, false>(a, tmKh, tmKl, st);
}

template <int D>
us_status launch_proxy_d(const ProxyArgs& a, const CUtensorMap& tmKh, const CUtensorMap& tmKl, cudaStream_t st) {
  switch (a.sw) {
    case 8: return launch_proxy_t<D, 8>(a, tmKh, tmKl, st);
    case 4: return launch_proxy_t<D, 4>(a, tmKh, tmKl, st);
    case 2: return launch_proxy_t<D, 2>(a, tmKh, tmKl, st);
    case 1: return launch_proxy_t<D, 1>(a, tmKh, tmKl, st);
    default:
      set_error("proxy: unsupported slot width");
      return US_ERR_UNSUPPORTED;
  }
}

}  // namespace

int proxy_slot_width(int rk) { return rk >= 8 ? 8 : rk; }

us_status launch_proxy(const ProxyArgs& a, const CUtensorMap& tmKh, const CUtensorMap& tmKl, cudaStream_t st) {
  if (a.rq > 128) {
    set_error("proxy: S/c_q above 128 unsupported");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_proxy_d<128>(a, tmKh, tmKl, st);
  if (a.D == 64) return launch_proxy_d<64>(a, tmKh, tmKl, st);
  set_error("proxy: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
