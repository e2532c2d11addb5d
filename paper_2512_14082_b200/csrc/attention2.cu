// attention2.cu — block-sparse FlashAttention forward, 128-key steps
// (reference block_sparse_attention, attention.cpp:89-137).
//
// Same semantics as attention.cu (ascending selected key blocks, token-level
// causality inside the diagonal block, online softmax, O = acc / den,
// lse = m + log den); different step shape:
//
// CTA = ONE UMMA M=128 tile = two 64-row query groups that read the same KV
// head. Its steps walk the ascending union of the two groups' selected blocks
// TWO blocks at a time: S = Q [K_a; K_b]^T is one M=128 x N=128 MMA chain
// (a 64-key tail step uses N=64), so every fixed per-step cost of the
// S -> softmax -> P.V round trip (TMEM load latency, P store, hand-offs) is
// paid once per 128 keys instead of once per 64 (attention.cu, r01d: ~3000
// cycles per 64-key step for 622 cycles of MMA). A group that did not select
// one of the two blocks gets -inf logits (P = 0) for its 64 columns.
//
// K tiles land by TMA in a K ring laid out chunk-major ([d-chunk][stage][64 keys]
// x 128 B), so the two stages of a step are contiguous and one SWIZZLE_128B
// descriptor covers N = 128 keys; V stays stage-major (P.V reads it 16 keys at
// a time). The ring has an even stage count and steps always take stages
// (2m, 2m+1), so a step never wraps.
//
// TMEM (448 of 512 columns): S0 [0,128), S1 [128,256) — S is double buffered,
// so S(k+1) runs on the tensor pipe while the softmax works on S(k); P (bf16x2)
// is aliased into the first 64 columns of its S buffer (TS-mode P.V), O
// [256, 256+D), Q [384, 384+D/2) (TS-mode S MMA). Issue order on the pipe:
// S0 S1 | PV0 S2 | PV1 S3 | ... — PV(k) precedes S(k+2) (which overwrites its
// S/P buffer) and S(k) completes after PV(k-2), so the softmax of step k only
// has to wait for PV(k-1) (bar_pvdone) before it rescales O.
//
// Roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warp 2 union-list builder, warp 3 idle, warps 4-7 softmax (thread = row,
// 128 key columns per step).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

constexpr int kBS = 64;
constexpr int kMaxN = 4096;
constexpr int kMaxW = kMaxN / 32;

template <int D>
struct Attn2Smem {
  static constexpr int kST = D == 128 ? 6 : 12;  // even: a step takes stages (2m, 2m+1)
  static constexpr int kChunks = D / 64;
  static constexpr int kTileBytes = kBS * 128;  // one 64-key x 64-element chunk (8 KB)
  static constexpr int kKBytes = kST * kChunks * kTileBytes;
  static constexpr int kVStage = kChunks * kTileBytes;
  static constexpr int kBytes = kKBytes + kST * kVStage;
  // K chunk kc of stage s (chunk-major: stages contiguous within a chunk)
  static constexpr int k_off(int kc, int s) { return (kc * kST + s) * kTileBytes; }
  static constexpr int v_off(int s) { return kKBytes + s * kVStage; }
};

constexpr uint32_t kTS0 = 0, kTO = 256, kTQ = 384;

#ifndef US_ATTN2_POLY_FROM
#define US_ATTN2_POLY_FROM 56
#endif
constexpr int kPolyFrom = US_ATTN2_POLY_FROM;  // columns [kPolyFrom, 64) of a full off-diagonal half

__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));  // 1.5 * 2^23
  const float2 n = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = __ffma2_rn(n, make_float2(-1.0f, -1.0f), x);
  float2 p = __ffma2_rn(make_float2(0.05508868396282196f, 0.05508868396282196f), f,
                        make_float2(0.24260404706001282f, 0.24260404706001282f));
  p = __ffma2_rn(p, f, make_float2(0.6932762265205383f, 0.6932762265205383f));
  p = __ffma2_rn(p, f, make_float2(0.9999289512634277f, 0.9999289512634277f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// Two query groups per CTA, KV head outermost, query blocks heaviest-first.
//   group_mode 0 / 1 (G even): heads (h, h+1) of one KV group at query block i
//   group_mode 2 (G odd):     one head at query blocks (i, i-1)
struct Pair {
  int b, h[2], i[2];
  bool en[2];
};

__device__ __forceinline__ Pair decode_pair(const AttnArgs& a, int item) {
  Pair g;
  if (a.group_mode != 2) {
    const int pairs = a.H / 2;
    const int i = a.N - 1 - item % a.N;
    const int bp = item / a.N;
    g.b = bp / pairs;
    const int h0 = (bp % pairs) * 2;
    g.h[0] = h0;
    g.h[1] = h0 + 1;
    g.i[0] = g.i[1] = i;
    g.en[0] = g.en[1] = true;
  } else {
    const int np = (a.N + 1) / 2;
    const int ip = np - 1 - item % np;
    const int bh = item / np;
    g.b = bh / a.H;
    g.h[0] = g.h[1] = bh % a.H;
    g.i[0] = 2 * ip + 1;
    g.i[1] = 2 * ip;
    g.en[0] = g.i[0] < a.N;
    g.en[1] = true;
  }
  return g;
}

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn2_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                 const AttnArgs a) {
  using SL = Attn2Smem<D>;
  constexpr int kST = SL::kST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_kvfull[kST], bar_kvempty[kST], bar_sfull[2], bar_pfull[2], bar_pvdone,
      bar_ofull;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int n_steps_sh;
  __shared__ uint32_t mrow[2][kMaxW];
  // ascending union of the two groups' selected blocks: j | sel_g << (16 + g)
  __shared__ uint32_t steps[kMaxN];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.H / a.H_kv;
  const Pair gr = decode_pair(a, blockIdx.x);
  const int kvh = gr.h[0] / G;
  int jmax = -1;
  for (int k = 0; k < 2; ++k)
    if (gr.en[k]) jmax = max(jmax, gr.i[k]);

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 4);
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kvfull[s], 1);
      mbar_init(&bar_kvempty[s], 1);
    }
    mbar_init(&bar_sfull[0], 1);
    mbar_init(&bar_sfull[1], 1);
    mbar_init(&bar_pfull[0], 4);
    mbar_init(&bar_pfull[1], 4);
    mbar_init(&bar_pvdone, 1);
    mbar_init(&bar_ofull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 2) {
    const int nw = jmax >= 0 ? (jmax >> 5) + 1 : 0;
    for (int g = 0; g < 2; ++g) {
      const int ig = gr.i[g];
      const uint32_t* src =
          a.mask ? a.mask + ((long long)(gr.b * a.planes + gr.h[g] / a.heads_per_plane) * a.N + ig) * a.W
                 : nullptr;
      for (int w = lane; w < nw; w += 32) {
        uint32_t word = 0;
        if (gr.en[g] && (w << 5) <= ig) {
          word = src ? src[w] : ~0u;
          const int hi = ig - (w << 5);
          if (hi < 31) word &= (2u << hi) - 1u;
        }
        mrow[g][w] = word;
      }
    }
    __syncwarp();
    int base = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int w = w0 + lane;
      const uint32_t m0 = w < nw ? mrow[0][w] : 0u, m1 = w < nw ? mrow[1][w] : 0u;
      uint32_t u = m0 | m1;
      const int cnt = __popc(u);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = base + incl - cnt;
      while (u) {
        const int bit = __ffs(u) - 1;
        u &= u - 1u;
        steps[pos++] = uint32_t((w << 5) + bit) | (((m0 >> bit) & 1u) << 16) | (((m1 >> bit) & 1u) << 17);
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) n_steps_sh = base;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int T = n_steps_sh;            // union positions
  const int nsteps = (T + 1) >> 1;     // 128-key steps (the last may hold one block)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t pol = policy_evict_last();
      const int kvrow0 = (gr.b * a.H_kv + kvh) * a.L;
      for (int t = 0; t < T; ++t) {
        const int j = int(steps[t] & 0xFFFFu);
        const int s = t % kST;
        if (t >= kST) mbar_wait(&bar_kvempty[s], ((t / kST) + 1) & 1);
        mbar_arrive_expect_tx(&bar_kvfull[s], 2 * SL::kChunks * SL::kTileBytes);
        for (int kc = 0; kc < SL::kChunks; ++kc) {
          tma_load_2d_hint(smem + SL::k_off(kc, s), &tmK, &bar_kvfull[s], kc * 64, kvrow0 + j * kBS, pol);
          tma_load_2d_hint(smem + SL::v_off(s) + kc * SL::kTileBytes, &tmV, &bar_kvfull[s], kc * 64,
                           kvrow0 + j * kBS, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s128 = idesc_f16(128, 128, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_s64 = idesc_f16(128, 64, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(128, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    auto issue_s = [&](int kk) {
      const int t0 = 2 * kk, s0 = t0 % kST;
      const bool two = t0 + 1 < T;
      mbar_wait(&bar_kvfull[s0], (t0 / kST) & 1);
      if (two) mbar_wait(&bar_kvfull[s0 + 1], ((t0 + 1) / kST) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d_tmem = tmem + kTS0 + (kk & 1) * 128;
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(smem_u32(smem + SL::k_off(kc, s0)) + ks * 32, 16, 1024);
            umma_f16_ts(d_tmem, tmem + kTQ + (kc * 4 + ks) * 8, bd, two ? idesc_s128 : idesc_s64,
                        (kc | ks) != 0);
          }
        umma_commit(&bar_sfull[kk & 1]);
      }
      __syncwarp();
    };
    mbar_wait(&bar_q, 0);
    tc_fence_after();
    if (nsteps > 0) issue_s(0);
    if (nsteps > 1) issue_s(1);
    for (int k = 0; k < nsteps; ++k) {
      const int t0 = 2 * k, s0 = t0 % kST;
      const bool two = t0 + 1 < T;
      mbar_wait(&bar_pfull[k & 1], (k >> 1) & 1);  // P(k) is in TMEM (aliased into S buffer k&1)
      tc_fence_after();
      if (elect_one()) {
        const uint32_t pbase = tmem + kTS0 + (k & 1) * 128;
        const int nks = two ? 8 : 4;
        for (int ks = 0; ks < nks; ++ks) {
          const int s = s0 + (ks >> 2);
          const uint64_t bd = sdesc_sw128(smem_u32(smem + SL::v_off(s)) + (ks & 3) * 16 * 128, kBS * 128, 1024);
          umma_f16_ts(tmem + kTO, pbase + ks * 8, bd, idesc_o, (k > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(&bar_kvempty[s0]);
        if (two) umma_commit(&bar_kvempty[s0 + 1]);
        umma_commit(&bar_pvdone);
      }
      __syncwarp();
      if (k + 2 < nsteps) issue_s(k + 2);
    }
    if (elect_one()) umma_commit(&bar_ofull);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int g = row >> 6, rloc = row & 63;
    const int ig = gr.i[g], hg = gr.h[g];
    const bool en = gr.en[g];
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const uint32_t tb = tmem + lane_addr;
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    bool started = false;
    {
      const uint4* src = reinterpret_cast<const uint4*>(
          a.Q + ((long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D);
#pragma unroll
      for (int c0 = 0; c0 < D / 2; c0 += 16) {
        uint32_t w16[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 v = en ? __ldg(src + c0 / 4 + u) : make_uint4(0, 0, 0, 0);
          w16[4 * u] = v.x;
          w16[4 * u + 1] = v.y;
          w16[4 * u + 2] = v.z;
          w16[4 * u + 3] = v.w;
        }
        tmem_st16(tb + kTQ + c0, w16);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_q);
    }
    for (int k = 0; k < nsteps; ++k) {
      const int t0 = 2 * k;
      const bool two = t0 + 1 < T;
      const uint32_t e0 = steps[t0], e1 = two ? steps[t0 + 1] : 0u;
      const bool sel0 = (e0 >> (16 + g)) & 1u, sel1 = two && ((e1 >> (16 + g)) & 1u);
      const bool diag0 = sel0 && int(e0 & 0xFFFFu) == ig, diag1 = sel1 && int(e1 & 0xFFFFu) == ig;
      const uint32_t sb = tb + kTS0 + (k & 1) * 128;
      mbar_wait(&bar_sfull[k & 1], (k >> 1) & 1);
      tc_fence_after();
      float sv[128];
      if (sel0 || sel1) {
        uint32_t* v = reinterpret_cast<uint32_t*>(sv);
        tmem_ld32(sb, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(sb + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_ld32(sb + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
        tmem_ld32(sb + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
        tmem_ld_wait();
      }
      uint32_t packed[64];
      if (sel0 || sel1) {
        // causal mask inside a diagonal block; -inf for a block this row's group did not select
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          if (!sel0 || (diag0 && c > rloc)) sv[c] = -INFINITY;
          if (!sel1 || (diag1 && c > rloc)) sv[64 + c] = -INFINITY;
        }
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = sv[u];
#pragma unroll
        for (int c = 8; c < 128; ++c) m8[c & 7] = fmaxf(m8[c & 7], sv[c]);
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        mx *= sl2;
        const bool need = mx > m_used + 8.f;
        const bool need_o = need && started;
        if (__any_sync(0xffffffffu, need_o)) {
          // O rescale once P.V(k-1) has retired (warp-collective TMEM ld/st; f = 1 for rows that did not move)
          if (k > 0) mbar_wait(&bar_pvdone, (k - 1) & 1);
          tc_fence_after();
          const float f = need_o ? ex2_approx(m_used - mx) : 1.f;
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tb + kTO + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            US_TMEM_ST_X32(tb + kTO + c0, o);
          }
          tmem_st_wait();
        }
        if (need) {
          if (started) l *= ex2_approx(m_used - mx);
          m_used = mx;
        }
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_used, -m_used);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool selh = h ? sel1 : sel0, diagh = h ? diag1 : diag0;
          if (!selh) {
#pragma unroll
            for (int c = 0; c < 32; ++c) packed[h * 32 + c] = 0u;
          } else if (!diagh) {
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float2 xx = __ffma2_rn(make_float2(sv[h * 64 + c], sv[h * 64 + c + 1]), sl2v, nm);
              float2 p;
              if (c >= kPolyFrom) {
                p = ex2_poly2(xx);
              } else {
                p.x = ex2_approx(xx.x);
                p.y = ex2_approx(xx.y);
              }
              acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
              packed[h * 32 + (c >> 1)] = pack_bf16(p.x, p.y);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              const float2 xx = __ffma2_rn(make_float2(sv[h * 64 + c], sv[h * 64 + c + 1]), sl2v, nm);
              float2 p;
              p.x = ex2_approx(xx.x);
              p.y = ex2_approx(xx.y);
              acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
              packed[h * 32 + (c >> 1)] = pack_bf16(p.x, p.y);
            }
          }
        }
        const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        l += s2.x + s2.y;
        started = true;
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) packed[c] = 0u;
      }
      // P -> TMEM columns [0, 64) of this S buffer (all S reads of this thread are done)
      {
        const uint32_t* p0 = packed;
        const uint32_t* p1 = packed + 32;
        US_TMEM_ST_X32(sb, p0);
        US_TMEM_ST_X32(sb + 32, p1);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[k & 1]);
    }
    // ---- epilogue
    mbar_wait(&bar_ofull, 0);
    tc_fence_after();
    const bool write = en && l > 0.f;
    const float inv_l = 1.f / l;
    __nv_bfloat16* dst = a.O + ((long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 16) {
      uint32_t o[16];
      tmem_ld16(tb + kTO + c0, o);
      tmem_ld_wait();
      if (write) {
        uint4 w0, w1;
        w0.x = pack_bf16(__uint_as_float(o[0]) * inv_l, __uint_as_float(o[1]) * inv_l);
        w0.y = pack_bf16(__uint_as_float(o[2]) * inv_l, __uint_as_float(o[3]) * inv_l);
        w0.z = pack_bf16(__uint_as_float(o[4]) * inv_l, __uint_as_float(o[5]) * inv_l);
        w0.w = pack_bf16(__uint_as_float(o[6]) * inv_l, __uint_as_float(o[7]) * inv_l);
        w1.x = pack_bf16(__uint_as_float(o[8]) * inv_l, __uint_as_float(o[9]) * inv_l);
        w1.y = pack_bf16(__uint_as_float(o[10]) * inv_l, __uint_as_float(o[11]) * inv_l);
        w1.z = pack_bf16(__uint_as_float(o[12]) * inv_l, __uint_as_float(o[13]) * inv_l);
        w1.w = pack_bf16(__uint_as_float(o[14]) * inv_l, __uint_as_float(o[15]) * inv_l);
        reinterpret_cast<uint4*>(dst + c0)[0] = w0;
        reinterpret_cast<uint4*>(dst + c0)[1] = w1;
      }
    }
    if (write && a.lse)
      a.lse[(long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + rloc] =
          (m_used + __log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int D>
us_status launch_attn2_t(const AttnArgs& a, const CUtensorMap& tmK, const CUtensorMap& tmV, cudaStream_t st) {
  const int smem = Attn2Smem<D>::kBytes + 1024;
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(attn2_kernel<D>, smem, attr_done, "attn2_kernel smem attribute"); s != US_OK)
    return s;
  long long items;
  if (a.group_mode != 2) items = (long long)a.B * (a.H / 2) * a.N;
  else items = (long long)a.B * a.H * ((a.N + 1) / 2);
  attn2_kernel<D><<<unsigned(items), 256, smem, st>>>(tmK, tmV, a);
  US_LAUNCH_CHECK("attn2_kernel");
  return US_OK;
}

}  // namespace

us_status launch_attention2(const AttnArgs& a, const CUtensorMap& tmK, const CUtensorMap& tmV, cudaStream_t st) {
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_attn2_t<128>(a, tmK, tmV, st);
  if (a.D == 64) return launch_attn2_t<64>(a, tmK, tmV, st);
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
