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
  static constexpr int kQ = 0;                         // [kc][128 rows][128 B]
  static constexpr int kQBytes = kBM * D * 2;
  static constexpr int kKVBytes = kBS * D * 2;         // one of K / V per stage
  static constexpr int kK = kQ + kQBytes;              // stage s: K at kK + s*2*kKVBytes, V after
  static constexpr int kP = kK + kST * 2 * kKVBytes;   // 2 x [128 rows][128 B]
  static constexpr int kPBytes = kBM * kBS * 2;
  static constexpr int kBytes = kP + 2 * kPBytes;
};

struct UnionIter {
  const uint32_t* m0;
  const uint32_t* m1;
  int w, wmax;
  uint32_t cur;
  __device__ void init(const uint32_t* a, const uint32_t* b, int jmax) {
    m0 = a;
    m1 = b;
    w = 0;
    wmax = jmax >> 5;
    cur = jmax >= 0 ? (a[0] | b[0]) : 0u;
  }
  __device__ bool next(int& j, bool& s0, bool& s1) {
    while (cur == 0u) {
      if (++w > wmax) return false;
      cur = m0[w] | m1[w];
    }
    const int bit = __ffs(cur) - 1;
    cur &= cur - 1u;
    j = (w << 5) + bit;
    s0 = (m0[w] >> bit) & 1u;
    s1 = (m1[w] >> bit) & 1u;
    return true;
  }
};

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using SL = AttnSmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_kvfull[kST], bar_kvempty[kST], bar_sfull[2], bar_sempty[2],
      bar_pfull[2], bar_pempty[2], bar_ofull;
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint32_t mrow[2][kMaxW];

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
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kvfull[s], 1);
      mbar_init(&bar_kvempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sempty[s], 4);
      mbar_init(&bar_pfull[s], 4);
      mbar_init(&bar_pempty[s], 1);
    }
    mbar_init(&bar_ofull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 256);
  if (warp == 2 || warp == 3) {
    // mask rows, restricted to the causal prefix j <= i_g
    const int g = warp - 2;
    const int ig = g ? i1 : i0;
    const bool en = g ? en1 : true;
    const int hg = g ? h1 : h0;
    const uint32_t* src = a.mask ? a.mask + ((long long)(b * a.planes + hg / a.heads_per_plane) * a.N + ig) * a.W : nullptr;
    for (int w = lane; w < kMaxW; w += 32) {
      uint32_t word = 0;
      if (en && w < a.W && (w << 5) <= ig) {
        word = src ? src[w] : ~0u;
        const int hi = ig - (w << 5);  // bits 0..hi are causal
        if (hi < 31) word &= (2u << hi) - 1u;
      }
      mrow[g][w] = word;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t tmem_o = tmem + 128;

  UnionIter it;
  it.init(mrow[0], mrow[1], jmax);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(&bar_q, SL::kQBytes);
      const int q0 = (b * a.H + h0) * a.L + i0 * kBS;
      const int q1 = (b * a.H + h1) * a.L + i1 * kBS;
      for (int kc = 0; kc < SL::kChunks; ++kc) {
        tma_load_2d(smem + SL::kQ + kc * kBM * 128, &tmQ, &bar_q, kc * 64, q0);
        tma_load_2d(smem + SL::kQ + kc * kBM * 128 + kBS * 128, &tmQ, &bar_q, kc * 64, q1);
      }
      int j, t = 0;
      bool s0, s1;
      const int kvrow0 = (b * a.H_kv + kvh) * a.L;
      while (it.next(j, s0, s1)) {
        const int s = t % kST;
        if (t >= kST) mbar_wait(&bar_kvempty[s], ((t / kST) + 1) & 1);
        uint8_t* sk = smem + SL::kK + s * 2 * SL::kKVBytes;
        uint8_t* sv = sk + SL::kKVBytes;
        mbar_arrive_expect_tx(&bar_kvfull[s], 2 * SL::kKVBytes);
        for (int kc = 0; kc < SL::kChunks; ++kc) {
          tma_load_2d_hint(sk + kc * kBS * 128, &tmK, &bar_kvfull[s], kc * 64, kvrow0 + j * kBS, pol_kv);
          tma_load_2d_hint(sv + kc * kBS * 128, &tmV, &bar_kvfull[s], kc * 64, kvrow0 + j * kBS, pol_kv);
        }
        ++t;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = idesc_f16(kBM, kBS, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(kBM, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    const uint32_t sQ = smem_u32(smem + SL::kQ);
    auto issue_pv = [&](int u) {
      const int pb = u & 1;
      mbar_wait(&bar_pfull[pb], (u >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sP = smem_u32(smem + SL::kP + pb * SL::kPBytes);
        const uint32_t sV = smem_u32(smem + SL::kK + (u % kST) * 2 * SL::kKVBytes + SL::kKVBytes);
#pragma unroll
        for (int ks = 0; ks < kBS / 16; ++ks) {
          const uint64_t ad = sdesc_sw128(sP + ks * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sV + ks * 16 * 128, kBS * 128, 1024);
          umma_f16_ss(tmem_o, ad, bd, idesc_o, (u > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(&bar_kvempty[u % kST]);
        umma_commit(&bar_pempty[pb]);
      }
      __syncwarp();
    };
    mbar_wait(&bar_q, 0);
    int j, t = 0;
    bool s0, s1;
    while (it.next(j, s0, s1)) {
      const int s = t % kST, sb = t & 1;
      mbar_wait(&bar_kvfull[s], (t / kST) & 1);
      if (t >= 2) mbar_wait(&bar_sempty[sb], ((t - 2) >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + SL::kK + s * 2 * SL::kKVBytes);
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad = sdesc_sw128(sQ + kc * kBM * 128 + ks * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sK + kc * kBS * 128 + ks * 32, 16, 1024);
            umma_f16_ss(tmem + sb * kBS, ad, bd, idesc_s, (kc | ks) != 0);
          }
        umma_commit(&bar_sfull[sb]);
      }
      __syncwarp();
      if (t >= 1) issue_pv(t - 1);
      ++t;
    }
    if (t >= 1) issue_pv(t - 1);
    if (elect_one()) umma_commit(&bar_ofull);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int g = row >> 6, rloc = row & 63;
    const int ig = g ? i1 : i0;
    const int hg = g ? h1 : h0;
    const bool en = g ? en1 : true;
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    uint8_t* sPbase = smem + SL::kP;
    int j, t = 0;
    bool s0, s1;
    while (it.next(j, s0, s1)) {
      const bool sel = g ? s1 : s0;
      const int sb = t & 1, pb = t & 1;
      mbar_wait(&bar_sfull[sb], (t >> 1) & 1);
      tc_fence_after();
      float sv[kBS];
      if (sel) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_addr + sb * kBS, v);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
        tmem_ld32(tmem + lane_addr + sb * kBS + 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[32 + c] = __uint_as_float(v[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sempty[sb]);

      uint32_t packed[kBS / 2];
      if (sel) {
        if (j == ig) {
#pragma unroll
          for (int c = 0; c < kBS; ++c)
            if (c > rloc) sv[c] = -INFINITY;
        }
        float mx = sv[0];
#pragma unroll
        for (int c = 1; c < kBS; ++c) mx = fmaxf(mx, sv[c]);
        mx *= sl2;
        const bool need = mx > m_used + 8.f;
        const bool need_o = need && l > 0.f;  // l > 0 implies t >= 1
        // tcgen05.ld/st are warp-collective (.sync.aligned): the O pass runs for
        // the whole warp whenever any of its rows moves its max; other rows use f = 1.
        if (__any_sync(0xffffffffu, need_o)) {
          const float f = need_o ? ex2_approx(m_used - mx) : 1.f;
          // previous P.V (step t-1) must have retired before touching O
          mbar_wait(&bar_pempty[(t - 1) & 1], ((t - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 16) {
            uint32_t o[16];
            tmem_ld16(tmem_o + lane_addr + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            tmem_st16(tmem_o + lane_addr + c0, o);
          }
          tmem_st_wait();
          l *= f;
        }
        if (need) m_used = mx;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < kBS; c += 2) {
          const float p0 = ex2_approx(fmaf(sv[c], sl2, -m_used));
          const float p1 = ex2_approx(fmaf(sv[c + 1], sl2, -m_used));
          sum += p0 + p1;
          packed[c >> 1] = pack_bf16(p0, p1);
        }
        l += sum;
      } else {
#pragma unroll
        for (int c = 0; c < kBS / 2; ++c) packed[c] = 0u;
      }
      if (t >= 2) mbar_wait(&bar_pempty[pb], ((t - 2) >> 1) & 1);
      uint8_t* sP = sPbase + pb * SL::kPBytes;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        *reinterpret_cast<uint4*>(sP + sw128_offset(row, ch)) =
            make_uint4(packed[4 * ch], packed[4 * ch + 1], packed[4 * ch + 2], packed[4 * ch + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[pb]);
      ++t;
    }
    mbar_wait(&bar_ofull, 0);
    tc_fence_after();
    if (en && t > 0) {
      const float inv_l = 1.f / l;
      __nv_bfloat16* dst = a.O + ((long long)(b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 16) {
        uint32_t o[16];
        tmem_ld16(tmem_o + lane_addr + c0, o);
        tmem_ld_wait();
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
      if (a.lse)
        a.lse[(long long)(b * a.H + hg) * a.L + (long long)ig * kBS + rloc] =
            (m_used + __log2f(l)) * 0.69314718055994531f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
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
  attn_kernel<D><<<unsigned(items), 256, smem, st>>>(tmQ, tmK, tmV, a);
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
