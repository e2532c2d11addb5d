// attention.cu — block-sparse FlashAttention forward on tcgen05/TMEM/TMA
// (SURVEY §8a-6).
//
// Reference: block_sparse_attention (attention.cpp:89-137): per head h and
// query block i, visit the selected key blocks j <= i in ascending order,
// tile = Q_i K_j^T / sqrt(d), strict-upper -inf inside the diagonal block,
// online softmax (running max, rescaled denominator and accumulator), then
// O = acc / den and lse = m + log(den).
//
// CTA = 4 "groups" (head, query block) that read the SAME KV head, as two
// UMMA M=128 tiles: tile A = groups 0,1 (rows 0-63 | 64-127), tile B = groups 2,3.
//   H/H_kv % 4 == 0 : 4 consecutive heads of a KV group at one query block
//   H/H_kv == 2     : both heads of the group at query blocks (i, i-1)
//   otherwise       : one head at 4 consecutive query blocks
// Every K/V tile staged in smem feeds up to 2 x 128 query rows (halving the
// L2->SM K/V traffic per FLOP of a 128-row design, which was the measured
// limit), and each tile only runs S/P.V for the union of ITS two groups'
// selected blocks; K/V is loaded for the union of all four. A group that did
// not select a block visited by its tile contributes P = 0 rows, so each
// group's output equals sparse attention over exactly its own selection.
//
// Roles (384 threads): warp 0 TMA producer (5-stage K/V ring), warps 1 / 3
// MMA issuers of tile A / B (warp 1 owns TMEM), warp 2 builds the union list
// (uint16 entries: block | slot bits << 12) and each tile's own-step list,
// warps 4-7 softmax of tile A, warps 8-11 softmax of tile B (thread = row).
// TMEM per tile X (256 cols at X*256): S [0,64) fp32, O [64,192), Q [192,256)
// (bf16x2, A operand of S = Q K^T, TS-mode MMA). P (bf16) goes to a
// 128 x 64 SWIZZLE_128B tile in SMEM and P.V is an SS-mode MMA, so the S
// columns are free as soon as the softmax has LOADED S(k): the issuer starts
// S(k+1) right then, and the tensor pipe computes the next logits while the
// softmax is still exponentiating — the S -> softmax -> P.V round trip no
// longer serialises each tile (r01d: the v6 step was ~3000 cycles for 622
// cycles of MMA). The issuer releases every union position in order (used ones
// by the P.V commit, skipped ones by a plain arrive); S(k+1) is issued early
// only when the next own position is < kST positions ahead, otherwise after
// P.V(k) (its ring stage may be the one P.V(k) frees).
// P.V(k) commits bar_pvdone: the softmax waits for P.V(k-1) before it
// overwrites the single P buffer or rescales O (both only touch state P.V(k-1)
// reads / writes; P.V(k-2) is always complete by then — it was issued before
// S(k) — so the parity wait is never more than one phase behind).
// Online softmax in log2 units with lazy rescaling: the running max used for
// exponentiation only moves when a row max exceeds it by > 8 (p <= 2^8).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"
#include "attn_common.cuh"

#ifndef US_ATTN_SKELETON
#define US_ATTN_SKELETON 0
#endif
// Debug timeline (tools/attn_trace.py): per step k of tile x of the traced CTA,
// clock64 at [S issued, S seen by softmax, P ready, P.V issued].
#ifndef US_ATTN_TRACE
#define US_ATTN_TRACE 0
#endif
#if US_ATTN_TRACE
__device__ long long g_attn_trace[2 * 4096 * 16];
__device__ int g_attn_trace_cta;
// (us_traced is computed once per thread at kernel entry: a per-event global load of
// g_attn_trace_cta cost the tracing warps hundreds of cycles per step)
#define TRACE(x, k, e)                                                                  \
  do {                                                                                  \
    if (us_traced && (k) < 4096) g_attn_trace[((x) * 4096 + (k)) * 16 + (e)] = clock64(); \
  } while (0)
#define TRACEV(x, k, e, v)                                                              \
  do {                                                                                  \
    if (us_traced && (k) < 4096) g_attn_trace[((x) * 4096 + (k)) * 16 + (e)] = (v); \
  } while (0)
#else
#define TRACEV(x, k, e, v) \
  do {                     \
  } while (0)
#define TRACE(x, k, e) \
  do {                 \
  } while (0)
#endif

// Calibration knob: 1 = skipped union positions are released by the TMA producer on behalf
// of the tile that skips them instead of by that tile's issuer when its own walk reaches
// them (a lagging tile then never holds ring stages it does not use). Measured neutral at
// C3 (profiles/r02c/README.md): the sparse step is bound by the selected group's softmax
// chain, not by the ring. Default 0 (the issuer walk).
#ifndef US_ATTN_PRODUCER_RELEASE
#define US_ATTN_PRODUCER_RELEASE 0
#endif

namespace us {
namespace {

using attn::kBS;
using attn::kMaxN;
using attn::kMaxW;
using attn::Groups;
using attn::decode_item;
using attn::ex2_poly2;

// K/V ring depth: a 64-key K+V tile takes ~1-2 us to land from L2, so the ring
// must cover several steps of prefetch.
// NT = tiles per CTA: 2 (one CTA per SM, the four groups share each K/V tile) or 1
// (two CTAs per SM, independent: no CTA waits on a shorter partner tile).
template <int D, int NT>
constexpr int stages_for() { return NT == 2 ? (D == 128 ? 5 : 10) : (D == 128 ? 2 : 4); }

template <int D, int NT = 2>
struct AttnSmem {
  static constexpr int kST = stages_for<D, NT>();
  static constexpr int kChunks = D / 64;
  static constexpr int kKVBytes = kBS * D * 2;       // one of K / V per stage
  static constexpr int kRingBytes = kST * 2 * kKVBytes;
  static constexpr int kPBytes = 128 * kBS * 2;      // per tile: 128 rows x 64 keys bf16
  static constexpr int kBytes = kRingBytes + NT * kPBytes;
};

// TMEM columns of tile X start at X * 256: S [0,64), O [64, 64+D), Q [192, 192+D/2).
constexpr uint32_t kTS = 0, kTO = 64, kTQ = 192;

#ifndef US_ATTN_POLY_FROM
#define US_ATTN_POLY_FROM 56
#endif
// columns [kPolyFrom, 64) of an off-diagonal tile use ex2_poly2 (FMA pipe)
constexpr int kPolyFrom = US_ATTN_POLY_FROM;

// One-tile CTAs: two groups that read the same KV head — two heads of a KV group at
// one query block (G even) or one head at query blocks (i, i-1) (G odd); groups 2, 3
// are disabled copies of group 0.
__device__ __forceinline__ Groups decode_pair(const AttnArgs& a, int item) {
  Groups g;
  const int G = a.H / a.H_kv;
  if (G % 2 == 0) {
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
  g.h[2] = g.h[3] = g.h[1];
  g.i[2] = g.i[3] = g.i[1];
  g.en[2] = g.en[3] = false;
  return g;
}

template <int D, int NT>
__global__ void __launch_bounds__(NT == 2 ? 384 : 192, NT == 2 ? 1 : 2)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using SL = AttnSmem<D, NT>;
  constexpr int kST = SL::kST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q[2], bar_kvfull[kST], bar_kvempty[kST], bar_sfull[2], bar_sfree[2], bar_pfull[2],
      bar_pvdone[2], bar_ofull[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ attn::Lists ls;
  __shared__ int kv_issued;  // union positions whose K/V load the producer has issued

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if US_ATTN_TRACE
  const bool us_traced = blockIdx.x == g_attn_trace_cta;
#endif
  const int G = a.H / a.H_kv;
  const Groups gr = NT == 2 ? decode_item(a, blockIdx.x) : decode_pair(a, blockIdx.x);
  const int kvh = gr.h[0] / G;
  if (a.sel_pairs && attn::m64_wins(a, gr.b, kvh)) return;  // sparse enough for attention64.cu (launched before)
  const int jmax = attn::last_block(a, gr);

  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(&bar_q[x], 4);
      mbar_init(&bar_sfull[x], 1);
      mbar_init(&bar_sfree[x], 4);
      mbar_init(&bar_pfull[x], 4);
      mbar_init(&bar_pvdone[x], 1);
    }
    for (int s = 0; s < kST; ++s) {
      mbar_init(&bar_kvfull[s], 1);
      mbar_init(&bar_kvempty[s], NT);
    }
    mbar_init(&bar_ofull[0], 1);
    mbar_init(&bar_ofull[1], 1);
    kv_issued = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, NT * 256);
  if (warp == 2) attn::build_lists(a, gr, jmax, NT == 2 && a.pairing, ls, ls.own_pos);
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
        // one 3-D TMA per tile: 64 rows x all d-chunks, landing as [chunk][row][128 B]
        tma_load_3d_hint(sk, &tmK, &bar_kvfull[s], 0, kvrow0 + j * kBS, 0, pol_kv);
        tma_load_3d_hint(sv, &tmV, &bar_kvfull[s], 0, kvrow0 + j * kBS, 0, pol_kv);
#if US_ATTN_PRODUCER_RELEASE
        // a tile that skips this position releases it right away (the producer arrives
        // for it); the issuers learn which loads exist from kv_issued
        for (int x = 0; x < NT; ++x)
          if (((ls.steps[t] >> (12 + 2 * x)) & 3u) == 0u) mbar_arrive(&bar_kvempty[s]);
        st_release_cta(&kv_issued, t + 1);
#endif
      }
    }
    __syncwarp();
  } else if (warp == 1 || (NT == 2 && warp == 3)) {
    // ------------------------------------------------------------ MMA issuers
    const int x = warp == 1 ? 0 : 1;
    constexpr uint32_t idesc_s = idesc_f16(128, kBS, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(128, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    const uint32_t tb = tmem + x * 256;
    const uint32_t sP = smem_u32(smem + SL::kRingBytes + x * SL::kPBytes);
    const int n_own = ls.n_own[x];
    // union position of own step kk (T past the last)
    auto own_at = [&](int kk) { return kk < n_own ? int(ls.own_pos[x][kk]) : T; };
    // Release union positions [from, to) this tile skips. Waiting for each tile to
    // land keeps this warp's kv_empty arrivals in phase order (one per stage phase).
    auto release = [&](int from, int to) {
#if US_ATTN_PRODUCER_RELEASE
      (void)from;
      (void)to;
#else
      for (int tt = from; tt < to; ++tt) {
        mbar_wait(&bar_kvfull[tt % kST], (tt / kST) & 1);
        if (lane == 0) mbar_arrive(&bar_kvempty[tt % kST]);
      }
#endif
    };
    auto issue_s = [&](int tt, int kk) {
      if (lane == 0) TRACE(x, kk, 7);  // issuer ready to issue S(kk)
#if US_ATTN_PRODUCER_RELEASE
      // Parity waits are only meaningful within one phase of a barrier, and this tile's
      // own positions can be far apart while the stage advances on positions it skips:
      // wait on kvfull(tt) only once the producer has ISSUED load tt, which implies load
      // tt - kST landed (its release needed it) — the barrier is at most one phase behind,
      // and it cannot be ahead (this tile still holds tt).
      while (ld_acquire_cta(&kv_issued) <= tt) __nanosleep(20);
#endif
      mbar_wait(&bar_kvfull[tt % kST], (tt / kST) & 1);
      if (lane == 0) TRACE(x, kk, 8);  // K/V of the step has landed
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
        umma_commit(&bar_sfull[x]);
        TRACE(x, kk, 0);
      }
      __syncwarp();
    };
    mbar_wait(&bar_q[x], 0);  // Q rows of tile x are in TMEM
    tc_fence_after();
    int t = own_at(0);
    release(0, t);
    if (t < T) issue_s(t, 0);
    int k = 0;
    while (t < T) {
      const int tn = own_at(k + 1);
      const bool early = tn < T && tn - t < kST;
      mbar_wait(&bar_sfree[x], k & 1);  // the softmax has loaded S(k): S columns are free
      if (lane == 0) TRACEV(x, k, 14, clock64());  // S(k) freed
      if (early) {
        release(t + 1, tn);
        issue_s(tn, k + 1);
      }
      mbar_wait(&bar_pfull[x], k & 1);  // P(k) is in SMEM
      if (lane == 0) TRACE(x, k, 9);     // all four warps' P(k) stored
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
        umma_commit(&bar_pvdone[x]);
        TRACE(x, k, 3);
      }
      __syncwarp();
      if (!early) {
        release(t + 1, tn);
        if (tn < T) issue_s(tn, k + 1);
      }
      t = tn;
      ++k;
    }
    if (elect_one()) umma_commit(&bar_ofull[x]);
    __syncwarp();
  } else if (warp >= (NT == 2 ? 4 : 2)) {
    // ------------------------------------------------------------ softmax / epilogue
    const int x = NT == 2 ? (warp - 4) >> 2 : 0;  // tile
    const int q = warp & 3;         // TMEM lane quarter
    const int row = q * 32 + lane;
    const int slot = 2 * x + (row >> 6), rloc = row & 63;
    const int g = int((ls.perm >> (2 * slot)) & 3u);
    const int ig = gr.i[g], hg = gr.h[g];
    const bool en = gr.en[g];
    const uint32_t lane_addr = uint32_t(q * 32) << 16;
    const uint32_t tb = tmem + lane_addr + x * 256;
    const uint32_t prow = smem_u32(smem + SL::kRingBytes + x * SL::kPBytes + row * 128);  // this row of the P tile
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    {
      // Q row -> TMEM (A operand of S = Q K^T: lane = row, 2 bf16 per column)
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
      if (lane == 0) mbar_arrive(&bar_q[x]);
    }
    int k = 0;
    const int n_own = ls.n_own[x];
    for (int kk = 0; kk < n_own; ++kk) {
      const uint32_t e = ls.steps[ls.own_pos[x][kk]];
      const int j = int(e & 0xFFFu);
      const bool sel = (e >> (12 + slot)) & 1u;
      mbar_wait(&bar_sfull[x], k & 1);
      tc_fence_after();
      if (row == 0) TRACE(x, k, 1);
      if (row == 0) TRACEV(x, k, 6, (long long)((e >> (12 + 2 * x)) & 3u));  // step kind
      float sv[kBS];
      if (sel) {
        uint32_t v[32], v2[32];
        tmem_ld32(tb + kTS, v);
        tmem_ld32(tb + kTS + 32, v2);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          sv[c] = __uint_as_float(v[c]);
          sv[32 + c] = __uint_as_float(v2[c]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_sfree[x]);  // S(k+1) may now overwrite the S columns
      if (row == 0) TRACE(x, k, 4);
      bool pv_prev_done = (k == 0);
      uint32_t packed[kBS / 2];
      if (sel) {
        const bool diag = (j == ig) && !a.noncausal;
        if (diag) {
#pragma unroll
          for (int c = 0; c < kBS; ++c)
            if (c > rloc) sv[c] = -INFINITY;
        }
        // exponentials against a given running max (log2 units) -> packed P row, row sum
        auto exps = [&](float m) {
          const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m, -m);
          float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
          if (!diag) {
#pragma unroll
            for (int c = 0; c < kBS; c += 2) {
              const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
              float2 p;
              if (c >= kPolyFrom) {
                p = ex2_poly2(xx);
              } else {
                p.x = ex2_approx(xx.x);
                p.y = ex2_approx(xx.y);
              }
              acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
              packed[c >> 1] = pack_bf16(p.x, p.y);
            }
          } else {
#pragma unroll
            for (int c = 0; c < kBS; c += 2) {
              const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
              float2 p;
              p.x = ex2_approx(xx.x);
              p.y = ex2_approx(xx.y);
              acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
              packed[c >> 1] = pack_bf16(p.x, p.y);
            }
          }
          const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
          const float2 s2 = __fadd2_rn(s01, s23);
          return s2.x + s2.y;
        };
        // 8 independent partial maxima (short dependency chains), then a tree
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(sv[u], fmaxf(sv[8 + u], sv[16 + u]));
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(sv[24 + u], sv[32 + u]));
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(sv[40 + u], fmaxf(sv[48 + u], sv[56 + u])));
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        mx *= sl2;
        const bool need = mx > m_used + 8.f;
        const bool need_o = need && l > 0.f;
        // O rescale (warp-collective TMEM ld/st) once P.V(k-1) has retired; rows
        // that did not move use f = 1.
        if (__any_sync(0xffffffffu, need_o)) {
          if (!pv_prev_done) {
            mbar_wait(&bar_pvdone[x], (k - 1) & 1);
            tc_fence_after();
            pv_prev_done = true;
          }
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
          l *= f;
        }
        if (need) m_used = mx;
        l += exps(m_used);
      } else {
#pragma unroll
        for (int c = 0; c < kBS / 2; ++c) packed[c] = 0u;
      }
      if (row == 0) TRACE(x, k, 5);
      // P(k) -> the SWIZZLE_128B P tile (row = 128 B = 8 chunks of 16 B); P.V(k-1)
      // must have consumed P(k-1) first
      if (!pv_prev_done) mbar_wait(&bar_pvdone[x], (k - 1) & 1);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        st_shared_v4(prow + ((c ^ (row & 7)) << 4), packed[4 * c], packed[4 * c + 1], packed[4 * c + 2],
                     packed[4 * c + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (row == 0) TRACE(x, k, 2);
      if (lane == 0) TRACE(x, k, 10 + q);  // this warp's P(k) hand-off
      if (lane == 0) mbar_arrive(&bar_pfull[x]);
      ++k;
    }
    // ---- epilogue
    mbar_wait(&bar_ofull[x], 0);
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
  if (warp == 1) tmem_dealloc(tmem, NT * 256);
}

template <int D, int NT>
us_status launch_attn_t(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                        const CUtensorMap& tmV, cudaStream_t st) {
  const int smem = AttnSmem<D, NT>::kBytes + 1024;  // + alignment slack
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(attn_kernel<D, NT>, smem, attr_done, "attn_kernel smem attribute"); s != US_OK)
    return s;
  long long items;
  if (NT == 1) {
    const int G = a.H / a.H_kv;
    items = G % 2 == 0 ? (long long)a.B * (a.H / 2) * a.N : (long long)a.B * a.H * ((a.N + 1) / 2);
  } else if (a.group_mode == 0) {
    items = (long long)a.B * (a.H / 4) * a.N;
  } else if (a.group_mode == 1) {
    items = (long long)a.B * a.H_kv * ((a.N + 1) / 2);
  } else {
    items = (long long)a.B * a.H * ((a.N + 3) / 4);
  }
  attn_kernel<D, NT><<<unsigned(items), NT == 2 ? 384 : 192, smem, st>>>(tmQ, tmK, tmV, a);
  US_LAUNCH_CHECK("attn_kernel");
  return US_OK;
}

}  // namespace

us_status launch_attention(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                           const CUtensorMap& tmV, cudaStream_t st) {
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
#ifdef US_CALIBRATION
  if (a.one_tile) {
    if (a.D == 128) return launch_attn_t<128, 1>(a, tmQ, tmK, tmV, st);
    if (a.D == 64) return launch_attn_t<64, 1>(a, tmQ, tmK, tmV, st);
  } else
#endif
  {
    if (a.D == 128) return launch_attn_t<128, 2>(a, tmQ, tmK, tmV, st);
    if (a.D == 64) return launch_attn_t<64, 2>(a, tmQ, tmK, tmV, st);
  }
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us

#if US_ATTN_TRACE
extern "C" int us_debug_attn_trace(int cta, long long* host_out) {
  if (host_out) return int(cudaMemcpyFromSymbol(host_out, ::g_attn_trace, sizeof(long long) * 2 * 4096 * 16));
  return int(cudaMemcpyToSymbol(::g_attn_trace_cta, &cta, sizeof(int)));
}
#endif
