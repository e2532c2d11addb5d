// attention.cu — block-sparse FlashAttention forward on tcgen05/TMEM/TMA
// (SURVEY §8a-6).
//
// Reference: block_sparse_attention (attention.cpp:89-137): per head h and
// query block i, visit the selected key blocks j <= i in ascending order,
// tile = Q_i K_j^T / sqrt(d), strict-upper -inf inside the diagonal block,
// online softmax (running max, rescaled denominator and accumulator), then
// O = acc / den and lse = m + log(den).
//
// CTA tile (M = 128 rows = one UMMA M):
//   rows   0..63  = group 0 = (head h0, query block i0)
//   rows  64..127 = group 1 = (head h1, query block i1)
// with both groups reading the SAME KV head, so every K/V tile staged in smem
// feeds both halves of one M=128 MMA (GQA head sharing). Pairing: heads
// (2p, 2p+1) of one KV group at the same query block when H/H_kv is even,
// else query blocks (2p, 2p+1) of one head. The CTA walks the ascending union
// of the two groups' selected blocks; a group that did not select block j
// contributes P = 0 rows (no exp work, no statistics update), so the output
// equals per-group sparse attention over exactly its own selected blocks.
//
// Roles (256 threads): warp 0 TMA producer (Q once, K/V ring of 4 stages),
// warp 1 MMA issuer and TMEM owner, warps 2-3 load the mask rows, warps 4-7
// softmax + epilogue (thread = row = TMEM lane).
// TMEM (256 cols): S double buffer [0,128) (2 x 64 fp32 cols), O [128,128+D).
// P goes registers -> bf16 -> 128B-swizzled smem (K-major A operand of P.V);
// V is the MN-major B operand straight from its row-major TMA tile.
// Online softmax in log2 units with lazy rescaling: the running max used for
// exponentiation only moves when a row max exceeds it by > 8 (p <= 2^8), and
// only then is the O row in TMEM rescaled (after the previous P.V retires).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

constexpr int kBM = 128;   // rows per CTA
constexpr int kBS = 64;    // block size (keys per tile, rows per group)
constexpr int kST = 4;     // K/V stages
constexpr int kMaxW = 128; // mask words per row (N <= 4096)

template <int D>
struct AttnSmem {
  static constexpr int kChunks = D / 64;
  static constexpr int kKVBytes = kBS * D * 2;         // one of K / V per stage
  static constexpr int kK = 0;                         // stage s: K at kK + s*2*kKVBytes, V after
  static constexpr int kBytes = kK + kST * 2 * kKVBytes;
};

// TMEM columns (512 allocated): S0 S1 | O0 | O1 | Q (bf16x2 packed) | P0 P1 (bf16x2 packed)
constexpr uint32_t kTS = 0, kTO = 128, kTQ = 384, kTP = 448;

// exp2 on the FMA/ALU pipes for a pair of values (offloads MUFU): round-to-nearest
// split x = n + f, f in [-0.5, 0.5], cubic minimax for 2^f (max rel. err 7.7e-5,
// far below the bf16 rounding of P), exponent added in the integer domain. x <= 8.
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

constexpr int kPolyFrom = 24;  // columns [24, 32) of a warpgroup half-tile use ex2_poly2 (25%)

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using SL = AttnSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_kvfull[kST], bar_kvempty[kST], bar_sfull[2], bar_sempty[2],
      bar_pfull[2], bar_pempty[2], bar_ofull;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int n_steps_sh;
  __shared__ uint32_t mrow[2][kMaxW];
  // union of the two groups' selected blocks, ascending: j | sel0 << 16 | sel1 << 17
  __shared__ uint32_t steps[kMaxW * 32];
  __shared__ float xm[2][kBM], xl[2][kBM];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.H / a.H_kv;

  // ---- work item (heavy query blocks first)
  int b, h0, h1, i0, i1;
  bool en1 = true;
  {
    const int item = blockIdx.x;
    if (a.pair_heads) {
      const int per_i = a.B * (a.H / 2);
      const int i = a.N - 1 - item / per_i;
      const int rem = item % per_i;
      b = rem / (a.H / 2);
      const int hp = rem % (a.H / 2);
      h0 = 2 * hp;
      h1 = h0 + 1;
      i0 = i1 = i;
    } else {
      const int npairs = (a.N + 1) / 2;
      const int per_ip = a.B * a.H;
      const int ip = npairs - 1 - item / per_ip;
      const int rem = item % per_ip;
      b = rem / a.H;
      h0 = h1 = rem % a.H;
      i0 = 2 * ip;
      i1 = i0 + 1;
      en1 = i1 < a.N;
    }
  }
  const int kvh = h0 / G;
  const int jmax = en1 ? max(i0, i1) : i0;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 4);
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kvfull[s], 1);
      mbar_init(&bar_kvempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sempty[s], 8);
      mbar_init(&bar_pfull[s], 8);
      mbar_init(&bar_pempty[s], 1);
    }
    mbar_init(&bar_ofull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 2) {
    // mask rows restricted to the causal prefix j <= i_g, then the ascending union list
    const int nw = (jmax >> 5) + 1;
    for (int g = 0; g < 2; ++g) {
      const int ig = g ? i1 : i0;
      const bool en = g ? en1 : true;
      const int hg = g ? h1 : h0;
      const uint32_t* src =
          a.mask ? a.mask + ((long long)(b * a.planes + hg / a.heads_per_plane) * a.N + ig) * a.W : nullptr;
      for (int w = lane; w < nw; w += 32) {
        uint32_t word = 0;
        if (en && (w << 5) <= ig) {
          word = src ? src[w] : ~0u;
          const int hi = ig - (w << 5);  // bits 0..hi are causal
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
  const int T = n_steps_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t pol_kv = policy_evict_last();
      const int kvrow0 = (b * a.H_kv + kvh) * a.L;
      for (int t = 0; t < T; ++t) {
        const int j = int(steps[t] & 0xFFFFu);
        const int s = t % kST;
        if (t >= kST) mbar_wait(&bar_kvempty[s], ((t / kST) + 1) & 1);
        uint8_t* sk = smem + SL::kK + s * 2 * SL::kKVBytes;
        uint8_t* sv = sk + SL::kKVBytes;
        mbar_arrive_expect_tx(&bar_kvfull[s], 2 * SL::kKVBytes);
        for (int kc = 0; kc < SL::kChunks; ++kc) {
          tma_load_2d_hint(sk + kc * kBS * 128, &tmK, &bar_kvfull[s], kc * 64, kvrow0 + j * kBS, pol_kv);
          tma_load_2d_hint(sv + kc * kBS * 128, &tmV, &bar_kvfull[s], kc * 64, kvrow0 + j * kBS, pol_kv);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // S(t) -> S buffer t&1; softmax warpgroup w turns columns [32w, 32w+32) of S(t)
    // into P(t) (P buffer t&1) with its own running max; O_w += P_w V_w. Event-driven:
    // S(t) is issued as soon as its K tile landed and S(t-2) was drained, P.V(t) as
    // soon as P(t) is complete — neither waits for the other.
    constexpr uint32_t idesc_s = idesc_f16(kBM, kBS, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(kBM, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    mbar_wait(&bar_q, 0);  // Q rows are in TMEM
    tc_fence_after();
    auto issue_s = [&](int t) {
      const int st = t % kST, sb = t & 1;
      mbar_wait(&bar_kvfull[st], (t / kST) & 1);
      if (t >= 2) mbar_wait(&bar_sempty[sb], ((t - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + SL::kK + st * 2 * SL::kKVBytes);
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(sK + kc * kBS * 128 + ks * 32, 16, 1024);
            umma_f16_ts(tmem + kTS + sb * kBS, tmem + kTQ + (kc * 4 + ks) * 8, bd, idesc_s, (kc | ks) != 0);
          }
        umma_commit(&bar_sfull[sb]);
      }
      __syncwarp();
    };
    // Fixed order with blocking waits: S(t+2) as soon as S(t) is drained (early in
    // softmax(t)), then P.V(t) once P(t) is complete (end of softmax(t)).
    if (T > 0) issue_s(0);
    if (T > 1) issue_s(1);
    for (int t = 0; t < T; ++t) {
      if (t + 2 < T) issue_s(t + 2);
      mbar_wait(&bar_pfull[t & 1], (t >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const int pb = t & 1;
        const uint32_t sV = smem_u32(smem + SL::kK + (t % kST) * 2 * SL::kKVBytes + SL::kKVBytes);
#pragma unroll
        for (int ks = 0; ks < kBS / 16; ++ks) {
          const int w = ks >> 1;  // keys [32w, 32w+32) belong to softmax warpgroup w
          const uint64_t bd = sdesc_sw128(sV + ks * 16 * 128, kBS * 128, 1024);
          umma_f16_ts(tmem + kTO + w * 128, tmem + kTP + pb * 32 + ks * 8, bd, idesc_o,
                      (t > 0 || (ks & 1)) ? 1u : 0u);
        }
        umma_commit(&bar_kvempty[t % kST]);
        umma_commit(&bar_pempty[pb]);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar_ofull);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    const int wg = (warp - 4) >> 2;  // softmax warpgroup = step parity it owns
    const int q = warp & 3;          // TMEM lane quarter
    const int row = q * 32 + lane;
    const int g = row >> 6, rloc = row & 63;
    const int ig = g ? i1 : i0;
    const int hg = g ? h1 : h0;
    const bool en = g ? en1 : true;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const uint32_t tS = tmem + lane_addr + kTS + wg * kBS;
    const uint32_t tO = tmem + lane_addr + kTO + wg * 128;
    const uint32_t tP = tmem + lane_addr + kTP + wg * 16;  // + 32 * (t & 1)
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    if (wg == 0) {
      // Q row -> TMEM (A operand of S = Q K^T: lane = row, 2 bf16 per column)
      const uint4* src = reinterpret_cast<const uint4*>(
          a.Q + ((long long)(b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D);
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
        tmem_st16(tmem + lane_addr + kTQ + c0, w16);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_q);
    }
    const uint32_t tShalf = tmem + lane_addr + kTS + wg * 32;
    for (int t = 0; t < T; ++t) {
      const uint32_t e = steps[t];
      const int j = int(e & 0xFFFFu);
      const bool sel = (e >> (16 + g)) & 1u;
      const int sb = t & 1;
      mbar_wait(&bar_sfull[sb], (t >> 1) & 1);
      tc_fence_after();
      float sv[32];
      if (sel) {
        uint32_t v[32];
        tmem_ld32(tShalf + sb * kBS, v);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sempty[sb]);
      // P buffer sb was last read by P.V(t-2)
      if (t >= 2) mbar_wait(&bar_pempty[sb], ((t - 2) >> 1) & 1);

      uint32_t packed[16];
      if (sel) {
        const bool diag = (j == ig);
        if (diag) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c + 32 * wg > rloc) sv[c] = -INFINITY;
        }
        float mx = fmaxf(sv[0], sv[1]);
#pragma unroll
        for (int c = 2; c < 32; c += 2) mx = fmaxf(mx, fmaxf(sv[c], sv[c + 1]));
        mx *= sl2;
        const bool need = mx > m_used + 8.f;
        const bool need_o = need && l > 0.f;
        // tcgen05.ld/st are warp-collective: the O pass runs for the whole warp
        // whenever any of its rows moves its max; other rows use f = 1.
        if (__any_sync(0xffffffffu, need_o)) {
          const float f = need_o ? ex2_approx(m_used - mx) : 1.f;
          // O_wg was last written by P.V(t-1)
          mbar_wait(&bar_pempty[(t - 1) & 1], ((t - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tO + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            US_TMEM_ST_X32(tO + c0, o);
          }
          tmem_st_wait();
          l *= f;
        }
        if (need) m_used = mx;
        // -inf (masked) when the warpgroup's half of this row has no live key yet
        const float mu = m_used == -INFINITY ? 0.f : m_used;
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-mu, -mu);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        if (!diag) {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
            float2 p;
            if (c >= kPolyFrom) {
              p = ex2_poly2(x);
            } else {
              p.x = ex2_approx(x.x);
              p.y = ex2_approx(x.y);
            }
            acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
            packed[c >> 1] = pack_bf16(p.x, p.y);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
            float2 p;
            p.x = ex2_approx(x.x);
            p.y = ex2_approx(x.y);
            acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
            packed[c >> 1] = pack_bf16(p.x, p.y);
          }
        }
        const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
        const float2 s2 = __fadd2_rn(s01, s23);
        l += s2.x + s2.y;
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) packed[c] = 0u;
      }
      tmem_st16(tP + sb * 32, packed);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[sb]);
    }
    // ---- merge the two warpgroups' partial softmax states (split over key steps)
    xm[wg][row] = m_used;
    xl[wg][row] = l;
    mbar_wait(&bar_ofull, 0);
    tc_fence_after();
    named_bar_sync(1, 256);
    const float m0 = xm[0][row], m1 = xm[1][row], l0 = xl[0][row], l1 = xl[1][row];
    const float mm = fmaxf(m0, m1);
    const float f0 = l0 > 0.f ? ex2_approx(m0 - mm) : 0.f;
    const float f1 = l1 > 0.f ? ex2_approx(m1 - mm) : 0.f;
    const float lt = l0 * f0 + l1 * f1;
    const float inv_l = 1.f / lt;
    const bool write = en && T > 0;
    __nv_bfloat16* dst = a.O + ((long long)(b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D;
    const uint32_t tO0 = tmem + lane_addr + kTO, tO1 = tO0 + 128;
#pragma unroll 1
    for (int c0 = wg * (D / 2); c0 < (wg + 1) * (D / 2); c0 += 16) {
      uint32_t o0[16], o1[16];
      tmem_ld16(tO0 + c0, o0);
      tmem_ld16(tO1 + c0, o1);
      tmem_ld_wait();
      float r[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float a0 = f0 > 0.f ? __uint_as_float(o0[c]) * f0 : 0.f;
        const float a1 = f1 > 0.f ? __uint_as_float(o1[c]) * f1 : 0.f;
        r[c] = (a0 + a1) * inv_l;
      }
      if (write) {
        uint4 w0, w1;
        w0.x = pack_bf16(r[0], r[1]);
        w0.y = pack_bf16(r[2], r[3]);
        w0.z = pack_bf16(r[4], r[5]);
        w0.w = pack_bf16(r[6], r[7]);
        w1.x = pack_bf16(r[8], r[9]);
        w1.y = pack_bf16(r[10], r[11]);
        w1.z = pack_bf16(r[12], r[13]);
        w1.w = pack_bf16(r[14], r[15]);
        reinterpret_cast<uint4*>(dst + c0)[0] = w0;
        reinterpret_cast<uint4*>(dst + c0)[1] = w1;
      }
    }
    if (write && wg == 0 && a.lse)
      a.lse[(long long)(b * a.H + hg) * a.L + (long long)ig * kBS + rloc] =
          (mm + __log2f(lt)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int D>
us_status launch_attn_t(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                        const CUtensorMap& tmV, cudaStream_t st) {
  const int smem = AttnSmem<D>::kBytes + 1024;
  static bool attr_set = false;
  if (!attr_set) {
    US_CUDA_TRY(cudaFuncSetAttribute(attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                "attn_kernel smem attribute");
    attr_set = true;
  }
  const long long items = a.pair_heads ? (long long)a.B * (a.H / 2) * a.N
                                       : (long long)a.B * a.H * ((a.N + 1) / 2);
  attn_kernel<D><<<unsigned(items), 384, smem, st>>>(tmQ, tmK, tmV, a);
  US_LAUNCH_CHECK("attn_kernel");
  return US_OK;
}

}  // namespace

us_status launch_attention(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                           const CUtensorMap& tmV, cudaStream_t st) {
  if (a.W > kMaxW) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_attn_t<128>(a, tmQ, tmK, tmV, st);
  if (a.D == 64) return launch_attn_t<64>(a, tmQ, tmK, tmV, st);
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
