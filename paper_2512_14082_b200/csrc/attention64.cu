// attention64.cu — block-sparse FlashAttention forward with one M = 64 UMMA chain per query
// group (the sparse-mask kernel).
//
// Reference: block_sparse_attention (attention.cpp:89-137): per head h and query block i,
// visit the selected key blocks j <= i in ascending order, tile = Q_i K_j^T / sqrt(d),
// strict-upper -inf inside the diagonal block, online softmax, O = acc / den,
// lse = m + log(den).
//
// attention.cu runs two 64-row query groups as one M = 128 tile over the UNION of their
// selections: with independent selections ~47 % of its rows are P = 0 at C3 and, worse,
// each SM holds only two step chains (one per tile) whose ~2 k-cycle softmax latency sets
// the pace (profiles/r02c). Here every query group is its own chain:
// * An M = 64 tcgen05 accumulator occupies TMEM lanes 0-15 of each 32-lane quarter (row
//   16 q + r in lane 32 q + r); with the accumulator / TMEM-A address at lane offset 16 it
//   occupies lanes 16-31 (profiles/r02c/m64_probes.txt). Two groups therefore share one set
//   of TMEM columns — S [0, 64), O [64, 64 + D), Q [192, 192 + D/2) — at lane offsets 0 and
//   16, and four groups (the CTA's work item, attn_common.cuh) fit in 512 columns.
// * An M = 64 MMA costs the cycles of an M = 128 one, so the tensor work per selected block
//   equals an M = 128 tile step, but no row is wasted on the other group's selection, and
//   each SM runs four independent chains instead of two.
// * Each group's softmax is four warps (one per lane quarter); a warp reads its 16 rows with
//   the 16x32bx2 TMEM shape — two threads per row, 32 key columns each; the row max is one
//   shuffle between the two.
// K/V tiles of 64 keys arrive by TMA once per union position (all four groups' selected
// blocks, ascending) into a ring shared by the four chains; the producer releases each
// position on behalf of the chains whose group skips it, so a chain only holds ring stages
// of its own positions.
//
// Warps (672 threads): 0 list builder + TMA producer, 1-3 and 20 MMA issuers of groups
// 0-3 (warp 1 owns TMEM), 4-19 softmax (warp 4 + 4 g + q: group g, lane quarter q).
#include "attn_common.cuh"
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

using attn::kBS;
using attn::kMaxN;

template <int D>
struct A64Smem {
  static constexpr int kST = D == 128 ? 5 : 10;  // K/V ring stages
  static constexpr int kChunks = D / 64;
  static constexpr int kKVBytes = kBS * D * 2;   // one of K / V per stage
  static constexpr int kRingBytes = kST * 2 * kKVBytes;
  static constexpr int kPBytes = 64 * kBS * 2;   // per group: 64 rows x 64 keys bf16, SWIZZLE_128B
  static constexpr int kBytes = kRingBytes + 4 * kPBytes;
};

constexpr uint32_t kTS = 0, kTO = 64, kTQ = 192;
constexpr int kThreads = 21 * 32;
constexpr int kPolyFrom = 28;  // columns >= this of each 32-column half of an off-diagonal block: FMA-pipe exp2

__device__ __forceinline__ int issuer_group(int warp) { return warp == 20 ? 3 : warp - 1; }

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn64_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const AttnArgs a) {
  using SL = A64Smem<D>;
  constexpr int kST = SL::kST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q[4], bar_kvfull[kST], bar_kvempty[kST], bar_sfull[4], bar_sfree[4], bar_pfull[4],
      bar_pvdone[4], bar_ofull[4];
  __shared__ uint32_t tmem_base_sh;
  __shared__ attn::ListsCore ls;
  __shared__ int kv_issued;  // union positions whose K/V load the producer has issued

  if (a.sel_pairs && !attn::m64_wins(a)) return;  // the mask is dense enough for attn_kernel
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.H / a.H_kv;
  attn::Groups gr;
  int kvh;
  if (a.items) {
    // four groups of one KV head with similar selected-block counts (attn64_items_kernel)
    const int per_kv = (G * a.N + 3) / 4;
    const int bk = int(blockIdx.x) / per_kv;
    gr.b = bk / a.H_kv;
    kvh = bk % a.H_kv;
    for (int k = 0; k < 4; ++k) {
      const int32_t e = a.items[(long long)blockIdx.x * 4 + k];
      gr.en[k] = e >= 0;
      gr.h[k] = e >= 0 ? (e >> 16) : kvh * G;
      gr.i[k] = e >= 0 ? (e & 0xFFFF) : 0;
    }
  } else {
    gr = attn::decode_item(a, blockIdx.x);
    kvh = gr.h[0] / G;
  }
  const int jmax = attn::last_block(a, gr);

  if (threadIdx.x == 32) {
    for (int g = 0; g < 4; ++g) {
      mbar_init(&bar_q[g], 4);
      mbar_init(&bar_sfull[g], 1);
      mbar_init(&bar_sfree[g], 4);
      mbar_init(&bar_pfull[g], 4);
      mbar_init(&bar_pvdone[g], 1);
      mbar_init(&bar_ofull[g], 1);
    }
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kvfull[s], 1);
      mbar_init(&bar_kvempty[s], 4);  // every chain releases every union position
    }
    kv_issued = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  // (no pairing: union bit 12 + g is group g)
  if (warp == 0) attn::build_lists(a, gr, jmax, false, ls, nullptr);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int T = ls.n_steps;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t pol_kv = policy_evict_last();
      const int kvrow0 = (gr.b * a.H_kv + kvh) * a.L;
      for (int t = 0; t < T; ++t) {
        const int j = int(ls.steps[t] & 0xFFFu);
        const int s = t % kST;
        if (t >= kST) mbar_wait(&bar_kvempty[s], ((t / kST) + 1) & 1);
        uint8_t* sk = smem + s * 2 * SL::kKVBytes;
        uint8_t* sv = sk + SL::kKVBytes;
        mbar_arrive_expect_tx(&bar_kvfull[s], 2 * SL::kKVBytes);
        tma_load_3d_hint(sk, &tmK, &bar_kvfull[s], 0, kvrow0 + j * kBS, 0, pol_kv);
        tma_load_3d_hint(sv, &tmV, &bar_kvfull[s], 0, kvrow0 + j * kBS, 0, pol_kv);
        // a chain whose group skips this position releases it right away (the producer
        // arrives for it): a chain only ever holds the stages of its own positions
        for (int g = 0; g < 4; ++g)
          if (((ls.steps[t] >> (12 + g)) & 1u) == 0u) mbar_arrive(&bar_kvempty[s]);
        *reinterpret_cast<volatile int*>(&kv_issued) = t + 1;
      }
    }
    __syncwarp();
  } else if (warp <= 3 || warp == 20) {
    // ------------------------------------------------------------ MMA issuer of group g
    const int g = issuer_group(warp);
    constexpr uint32_t idesc_s = idesc_f16(64, kBS, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(64, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    const uint32_t tb = tmem + (g >> 1) * 256 + (uint32_t((g & 1) * 16) << 16);
    const uint32_t sP = smem_u32(smem + SL::kRingBytes + g * SL::kPBytes);
    // next union position at or after p that group g selected (T past the last)
    auto own_from = [&](int p) {
      while (p < T && ((ls.steps[p] >> (12 + g)) & 1u) == 0u) ++p;
      return p;
    };
    // K/V of own position tt: a parity wait is only meaningful within one phase of the
    // barrier, and the stage advances on positions this chain skips, so the chain waits on
    // kvfull(tt) only once the producer has ISSUED load tt — which implies load tt - kST has
    // landed (its release needed it); the barrier cannot be ahead (this chain holds tt).
    auto wait_kv = [&](int tt) {
      while (*reinterpret_cast<const volatile int*>(&kv_issued) <= tt) __nanosleep(20);
      mbar_wait(&bar_kvfull[tt % kST], (tt / kST) & 1);
    };
    auto issue_s = [&](int tt) {
      wait_kv(tt);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + (tt % kST) * 2 * SL::kKVBytes);
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(sK + kc * kBS * 128 + ks * 32, 16, 1024);
            umma_f16_ts(tb + kTS, tb + kTQ + (kc * 4 + ks) * 8, bd, idesc_s, (kc | ks) != 0);
          }
        umma_commit(&bar_sfull[g]);
      }
      __syncwarp();
    };
    mbar_wait(&bar_q[g], 0);  // Q rows of group g are in TMEM
    tc_fence_after();
    int t = own_from(0);
    if (t < T) issue_s(t);
    int k = 0;
    while (t < T) {
      const int tn = own_from(t + 1);
      // S(k+1) early (right after the softmax has loaded S(k)) only when tn lies within kST
      // positions of t: its stage then last held a position before t, which every chain
      // has released or will release without waiting on this one (no cycle of chains
      // waiting on each other's P.V); otherwise after P.V(k)
      mbar_wait(&bar_sfree[g], k & 1);
      // ... or, further ahead, when its K/V has already landed (a non-blocking probe: a
      // chain never blocks on a stage before its own P.V(k) could free one)
      const bool early =
          tn < T && (tn - t < kST || (*reinterpret_cast<const volatile int*>(&kv_issued) > tn &&
                                      mbar_test_wait(&bar_kvfull[tn % kST], (tn / kST) & 1)));
      if (early) issue_s(tn);
      mbar_wait(&bar_pfull[g], k & 1);  // P(k) of the group's 64 rows is in SMEM
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sV = smem_u32(smem + (t % kST) * 2 * SL::kKVBytes + SL::kKVBytes);
#pragma unroll
        for (int ks = 0; ks < kBS / 16; ++ks) {
          const uint64_t ad = sdesc_sw128(sP + ks * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sV + ks * 16 * 128, kBS * 128, 1024);
          umma_f16_ss(tb + kTO, ad, bd, idesc_o, (k > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(&bar_kvempty[t % kST]);
        umma_commit(&bar_pvdone[g]);
      }
      __syncwarp();
      if (!early && tn < T) issue_s(tn);
      t = tn;
      ++k;
    }
    if (elect_one()) umma_commit(&bar_ofull[g]);
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int g = (warp - 4) >> 2;    // query group
    const int q = warp & 3;           // TMEM lane quarter (warp 4 + 4 g + q)
    const int half = lane >> 4;       // key columns [32 half, 32 half + 32), O columns [D/2 half, ...)
    const int r = 16 * q + (lane & 15);  // row of the group (0..63)
    const int ig = gr.i[g], hg = gr.h[g];
    const bool en = gr.en[g];
    // 16x32bx2 accesses of this warp's 16 lanes of group g
    const uint32_t tl = tmem + (g >> 1) * 256 + (uint32_t(32 * q + (g & 1) * 16) << 16);
    const uint32_t prow = smem_u32(smem + SL::kRingBytes + g * SL::kPBytes + r * 128);  // row r of the P tile
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;  // l: this thread's half of the row sum
    {
      // this half of the Q row -> TMEM (A operand of S = Q K^T, 2 bf16 per column)
      const uint4* src = reinterpret_cast<const uint4*>(
          a.Q + ((long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + r) * D);
#pragma unroll
      for (int c0 = 0; c0 < D / 4; c0 += 16) {
        uint32_t w16[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 v = en ? __ldg(src + (half * (D / 4) + c0) / 4 + u) : make_uint4(0, 0, 0, 0);
          w16[4 * u] = v.x;
          w16[4 * u + 1] = v.y;
          w16[4 * u + 2] = v.z;
          w16[4 * u + 3] = v.w;
        }
        tmem_st_16x32bx2_x16<D / 4>(tl + kTQ + c0, w16);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_q[g]);
    }
    auto own_from = [&](int p) {
      while (p < T && ((ls.steps[p] >> (12 + g)) & 1u) == 0u) ++p;
      return p;
    };
    int k = 0;
    int t = own_from(0);
    while (t < T) {
      const int j = int(ls.steps[t] & 0xFFFu);
      const int tn = own_from(t + 1);  // (independent shared loads: overlap the wait below)
      mbar_wait(&bar_sfull[g], k & 1);
      tc_fence_after();
      float sv[32];
      {
        uint32_t v[32];
        tmem_ld_16x32bx2_x32<32>(tl + kTS, v);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sfree[g]);  // S(k+1) may now overwrite the S columns
      bool pv_prev_done = (k == 0);
      const bool diag = (j == ig) && !a.noncausal;
      if (diag) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (32 * half + c > r) sv[c] = -INFINITY;
      }
      float m8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) m8[u] = fmaxf(fmaxf(sv[u], sv[8 + u]), fmaxf(sv[16 + u], sv[24 + u]));
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16)) * sl2;  // the row's other half
      // lazy rescale: the running max only moves when a row max exceeds it by > 8 (log2);
      // both threads of a row see the same mx, hence take the same decision
      const bool need = mx > m_used + 8.f;
      const bool need_o = need && m_used != -INFINITY;
      if (__any_sync(0xffffffffu, need_o)) {
        // O holds every key before this step once P.V(k-1) has retired; warp-collective
        // TMEM ld/st of this thread's half of the O columns, f = 1 for rows that did not move
        if (!pv_prev_done) {
          mbar_wait(&bar_pvdone[g], (k - 1) & 1);
          tc_fence_after();
          pv_prev_done = true;
        }
        const float f = need_o ? ex2_approx(m_used - mx) : 1.f;
#pragma unroll 1
        for (int c0 = 0; c0 < D / 2; c0 += 32) {
          uint32_t o[32];
          tmem_ld_16x32bx2_x32<D / 2>(tl + kTO + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
          tmem_st_16x32bx2_x32<D / 2>(tl + kTO + c0, o);
        }
        tmem_st_wait();
        l *= f;
      }
      if (need) m_used = mx;
      // exponentials of this thread's 32 columns -> packed bf16 pairs, row-sum half
      uint32_t packed[16];
      {
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_used, -m_used);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
          float2 p;
          if (c >= kPolyFrom && !diag) {  // (warp-uniform: both halves, 8 of 64 columns)
            p = attn::ex2_poly2(xx);
          } else {
            p.x = ex2_approx(xx.x);
            p.y = ex2_approx(xx.y);
          }
          acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
          packed[c >> 1] = pack_bf16(p.x, p.y);
        }
        const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        l += s2.x + s2.y;
      }
      // P(k) -> the group's SWIZZLE_128B P tile (row r: 8 chunks of 16 B, this thread's 4);
      // P.V(k-1) must have consumed P(k-1) first
      if (!pv_prev_done) mbar_wait(&bar_pvdone[g], (k - 1) & 1);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        st_shared_v4(prow + (((4 * half + c) ^ (r & 7)) << 4), packed[4 * c], packed[4 * c + 1], packed[4 * c + 2],
                     packed[4 * c + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[g]);
      t = tn;
      ++k;
    }
    // ---- epilogue: the row sum of both halves, this half of the O columns
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    mbar_wait(&bar_ofull[g], 0);
    tc_fence_after();
    const bool write = en && l > 0.f;
    const float inv_l = 1.f / l;
    __nv_bfloat16* dst = a.O + ((long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + r) * D + half * (D / 2);
#pragma unroll 1
    for (int c0 = 0; c0 < D / 2; c0 += 32) {
      uint32_t o[32];
      tmem_ld_16x32bx2_x32<D / 2>(tl + kTO + c0, o);
      tmem_ld_wait();
      if (write) {
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l);
          w.y = pack_bf16(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l);
          w.z = pack_bf16(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l);
          w.w = pack_bf16(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l);
          *reinterpret_cast<uint4*>(dst + c0 + c) = w;
        }
      }
    }
    if (write && a.lse && half == 0)
      a.lse[(long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + r] = (m_used + __log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// Selected key blocks j <= i of every mask row (one warp per row, lanes over the row's
// words), and their total over the heads (a.sel_pairs, the density gate's input).
__global__ void __launch_bounds__(256) attn64_counts_kernel(AttnArgs a) {
  __shared__ unsigned part[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rows = (long long)a.B * a.planes * a.N;
  const long long r = (long long)blockIdx.x * 8 + warp;
  unsigned n = 0;
  if (r < rows) {
    const int i = int(r % a.N);
    const uint32_t* row = a.mask + r * a.W;
    for (int w = lane; w <= (i >> 5); w += 32) {
      uint32_t word = row[w];
      const int hi = i - (w << 5);
      if (hi < 31) word &= (2u << hi) - 1u;
      n += __popc(word);
    }
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) a.row_counts[r] = int32_t(n);
  }
  if (a.sel_pairs) {
    if (lane == 0) part[warp] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int k = 0; k < 8; ++k) t += part[k];
      if (t) atomicAdd(a.sel_pairs, t * (unsigned long long)a.heads_per_plane);
    }
  }
}

// Work items for the four chains of a CTA: the G * N query groups of one (batch, KV head),
// ordered by their number of selected key blocks (heaviest first, counting sort), packed
// four at a time — so a CTA's chains have near-equal lengths (a CTA lasts as long as its
// longest chain: with four heads of one query block per CTA the longest is 1.33x the mean
// at C3, gain 8). One CTA per (batch, KV head); KV heads stay outermost in the grid order,
// so resident CTAs still share one KV head's K/V in L2.
__global__ void __launch_bounds__(1024) attn64_items_kernel(AttnArgs a) {
  extern __shared__ int hist[];  // [N + 2]: count histogram, then descending starts
  const int G = a.H / a.H_kv, N = a.N;
  const int bk = blockIdx.x, b = bk / a.H_kv, kvh = bk % a.H_kv;
  const int per_kv = (G * N + 3) / 4;
  int32_t* out = a.items + (long long)bk * per_kv * 4;
  for (int c = threadIdx.x; c < N + 2; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  auto count_of = [&](int e) {  // group e = (head kvh * G + e / N, query block e % N)
    const int h = kvh * G + e / N;
    return int(a.row_counts[(long long)(b * a.planes + h / a.heads_per_plane) * N + e % N]);
  };
  for (int e = threadIdx.x; e < G * N; e += blockDim.x) atomicAdd(&hist[count_of(e)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {  // descending exclusive starts (counts 0..N)
    int run = 0;
    for (int c = N; c >= 0; --c) {
      const int v = hist[c];
      hist[c] = run;
      run += v;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * N; e += blockDim.x) {
    const int pos = atomicAdd(&hist[count_of(e)], 1);
    out[pos] = ((kvh * G + e / N) << 16) | (e % N);
  }
  for (int pos = G * N + threadIdx.x; pos < per_kv * 4; pos += blockDim.x) out[pos] = -1;
}

template <int D>
us_status launch_a64_t(const AttnArgs& a, const CUtensorMap& tmK, const CUtensorMap& tmV, cudaStream_t st) {
  const int smem = A64Smem<D>::kBytes + 1024;  // + alignment slack
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(attn64_kernel<D>, smem, attr_done, "attn64_kernel smem attribute"); s != US_OK)
    return s;
  long long items = attn::work_items(a);
  if (a.items) {
    if (a.sel_pairs) US_CUDA_TRY(cudaMemsetAsync(a.sel_pairs, 0, sizeof(unsigned long long), st), "sel_pairs reset");
    const long long rows = (long long)a.B * a.planes * a.N;
    attn64_counts_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(a);
    US_LAUNCH_CHECK("attn64_counts_kernel");
    attn64_items_kernel<<<unsigned(a.B * a.H_kv), 1024, (a.N + 2) * 4, st>>>(a);
    US_LAUNCH_CHECK("attn64_items_kernel");
    items = (long long)a.B * a.H_kv * ((a.H / a.H_kv * a.N + 3) / 4);
  }
  attn64_kernel<D><<<unsigned(items), kThreads, smem, st>>>(tmK, tmV, a);
  US_LAUNCH_CHECK("attn64_kernel");
  return US_OK;
}

}  // namespace

long long attention64_item_entries(int B, int H, int H_kv, int N) {
  return (long long)B * H_kv * ((H / H_kv * N + 3) / 4) * 4;
}

size_t attention64_ws_bytes(int B, int H, int H_kv, int N) {
  return 4 * size_t(attention64_item_entries(B, H, H_kv, N)) + 16 + 4 * size_t(B) * H * N;
}

us_status launch_attention64(const AttnArgs& a, const CUtensorMap& tmK, const CUtensorMap& tmV, cudaStream_t st) {
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_a64_t<128>(a, tmK, tmV, st);
  if (a.D == 64) return launch_a64_t<64>(a, tmK, tmV, st);
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
