// attention_tp.cu — block-sparse FlashAttention forward on tcgen05/TMEM/TMA with
// P held in TMEM and the logits double-buffered.
//
// Reference: block_sparse_attention (attention.cpp:89-137): per head h and query
// block i, visit the selected key blocks j <= i in ascending order, tile =
// Q_i K_j^T / sqrt(d), strict-upper -inf inside the diagonal block, online
// softmax, O = acc / den, lse = m + log(den). dense_attention (attention.cpp:20-54)
// is the same walk over every (causal) block.
//
// CTA = 4 query groups (head, query block, 64 rows each) that read the same KV
// head, as two UMMA M = 128 tiles (attn_common.cuh: decode, union list, pairing).
// K/V tiles of 64 keys arrive once per union position through a TMA ring and
// feed both tiles.
//
// The softmax is taken out of the MMA chain:
// * Each tile has TWO logit buffers in TMEM. S(k+1) is computed while the softmax
//   works on S(k); P(k) is written back (bf16) into the columns of S(k) and
//   P.V(k) is a TS-mode MMA (A = P from TMEM, B = V from SMEM) that runs while the
//   softmax works on S(k+1). The issuer puts S(k+2) into the same buffer right
//   after P.V(k) (same issuing thread: the tensor pipe executes them in order, so
//   S(k+2) overwrites P(k) only after P.V(k) read it). In steady state the
//   softmax warps never wait for an MMA; the tensor pipe sees S and P.V of both
//   tiles back to back.
// * To fit two logit buffers per tile into the 512 TMEM columns, Q stays in SMEM
//   (TMA, once per CTA) and S = Q K^T is an SS-mode MMA.
// * Two softmax warps per TMEM lane quarter per tile (16 softmax warps): warp
//   half h owns key columns [32h, 32h + 32) of its 32 rows. The halves agree on
//   the row max through one shared-memory exchange per step (a 64-thread named
//   barrier); the running max only moves when a row max exceeds it by > 8 (log2
//   units) — then O is rescaled, after waiting for P.V(k-1), each half its own
//   half of the O columns. Row sums are kept per half and added in the epilogue.
//
// TMEM per tile X (256 columns at X * 256): S buffer b at [64 b, 64 b + 64) fp32,
// P (bf16x2) of key half h written at [64 b + 32 h, + 16) — inside the S columns
// that half itself loaded; O [128, 128 + D).
// SMEM: Q of tile X [D/64 chunks][128 rows][128 B] (SW128, K-major A operand), then
// the K/V ring. Warps (640 threads): 0 TMA producer, 1 / 3 MMA issuers of tile A /
// B (warp 1 owns TMEM), 2 list builder, 4-11 softmax of tile A, 12-19 of tile B.
#include "attn_common.cuh"
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

// Debug timeline (tools/tp_trace.py, tools/build_tp_trace.sh): clock64 per (tile, step, event)
// of one CTA. Events: 0 S issued, 12 K landed (issuer), 1/8 S seen (half 0/1, quarter 0),
// 2 S loaded, 3/9 max exchanged, 4 exps done, 5/10/11 P arrived (h0q0/h1q0/h0q3),
// 6 P seen by the issuer, 7 P.V issued.
#ifndef US_TP_TRACE
#define US_TP_TRACE 0
#endif
#if US_TP_TRACE
__device__ long long g_tp_trace[2 * 4096 * 16];
__device__ int g_tp_trace_cta;
#define TPTRACE(cond, x, k, e)                                                                     \
  do {                                                                                             \
    if (tp_traced && (cond) && (k) < 4096) g_tp_trace[((x) * 4096 + (k)) * 16 + (e)] = clock64(); \
  } while (0)
#else
#define TPTRACE(cond, x, k, e) \
  do {                         \
  } while (0)
#endif

namespace us {
namespace {

using attn::kBS;
using attn::kMaxN;

template <int D>
struct TpSmem {
  static constexpr int kChunks = D / 64;
  static constexpr int kQTile = 128 * D * 2;      // Q of one tile
  static constexpr int kTileBytes = kBS * D * 2;  // one K or V tile (64 keys)
#ifndef US_TP_SK
#define US_TP_SK 4
#endif
#ifndef US_TP_SV
#define US_TP_SV 4
#endif
  static constexpr int kSK = D == 128 ? US_TP_SK : 2 * US_TP_SK;  // K ring stages (released when S completes)
  static constexpr int kSV = D == 128 ? US_TP_SV : 2 * US_TP_SV;  // V ring stages (released when P.V completes)
  static constexpr int kKRing = 2 * kQTile;
  static constexpr int kVRing = kKRing + kSK * kTileBytes;
  static constexpr int kBytes = kVRing + kSV * kTileBytes;
};

constexpr uint32_t kTO = 128;
constexpr int kThreads = 640;

#ifndef US_TP_POLY
#define US_TP_POLY 6
#endif
// columns [32 - kPoly, 32) of each off-diagonal half row use ex2_poly2 (FMA pipe)
constexpr int kPoly = US_TP_POLY;

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using SL = TpSmem<D>;
  constexpr int kSK = SL::kSK, kSV = SL::kSV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q[2], bar_kfull[kSK], bar_kempty[kSK], bar_vfull[kSV], bar_vempty[kSV], bar_sfull[2][2],
      bar_pfull[2][2], bar_pvdone[2], bar_ofull[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ attn::ListsCore ls;
  // row-max exchange between the two key halves of a row, double-buffered by step parity
  __shared__ float xch[2][2][128][2];
  __shared__ float xl[2][128][2];  // row-sum exchange (epilogue)
  // union positions whose K / V load the producers have issued (published for the issuers)
  __shared__ int k_issued, v_issued;

  const int warp = threadIdx.x >> 5;
#if US_TP_TRACE
  const bool tp_traced = blockIdx.x == g_tp_trace_cta;
#endif
  const int G = a.H / a.H_kv;
  const attn::Groups gr = attn::decode_item(a, blockIdx.x);
  const int kvh = gr.h[0] / G;
  const int jmax = attn::last_block(a, gr);

  if (threadIdx.x == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(&bar_q[x], 1);
      mbar_init(&bar_sfull[x][0], 1);
      mbar_init(&bar_sfull[x][1], 1);
      // one P barrier per buffer: a softmax warp may finish step k + 1 before another
      // finishes step k, so the arrivals of consecutive steps must not share a barrier
      mbar_init(&bar_pfull[x][0], 8);
      mbar_init(&bar_pfull[x][1], 8);
      mbar_init(&bar_pvdone[x], 1);
      mbar_init(&bar_ofull[x], 1);
    }
    for (int s = 0; s < kSK; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], 2);
    }
    for (int s = 0; s < kSV; ++s) {
      mbar_init(&bar_vfull[s], 1);
      mbar_init(&bar_vempty[s], 2);
    }
    k_issued = 0;
    v_issued = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  if (warp == 2) attn::build_lists(a, gr, jmax, a.pairing != 0, ls, nullptr);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int T = ls.n_steps;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      // Q of both tiles: slot s (tile s / 2, rows (s & 1) * 64) holds group perm[s];
      // one 2-D box (64 rows x 64 elements) per (slot, chunk)
      const uint64_t pol_q = policy_evict_first();
      for (int x = 0; x < 2; ++x) {
        mbar_arrive_expect_tx(&bar_q[x], SL::kQTile);
        for (int r = 0; r < 2; ++r) {
          const int g = int((ls.perm >> (2 * (2 * x + r))) & 3u);
          // disabled groups (query block past N) load block 0 of their head: rows never used
          const int qrow = (gr.b * a.H + gr.h[g]) * a.L + (gr.en[g] ? gr.i[g] : 0) * kBS;
          for (int kc = 0; kc < SL::kChunks; ++kc)
            tma_load_2d_hint(smem + x * SL::kQTile + kc * 128 * 128 + r * 64 * 128, &tmQ, &bar_q[x], kc * 64, qrow,
                             pol_q);
        }
      }
      const uint64_t pol_kv = policy_evict_last();
      const int kvrow0 = (gr.b * a.H_kv + kvh) * a.L;
      for (int t = 0; t < T; ++t) {
        const int j = int(ls.steps[t] & 0xFFFu);
        const int s = t % kSK;
        if (t >= kSK) mbar_wait(&bar_kempty[s], ((t / kSK) + 1) & 1);
        mbar_arrive_expect_tx(&bar_kfull[s], SL::kTileBytes);
        // one 3-D TMA per tile: 64 rows x all d-chunks, landing as [chunk][row][128 B]
        tma_load_3d_hint(smem + SL::kKRing + s * SL::kTileBytes, &tmK, &bar_kfull[s], 0, kvrow0 + j * kBS, 0,
                         pol_kv);
        // a tile that skips this union position releases it right away: the producer
        // arrives for it, so no tile ever waits on loads it does not use
        for (int x = 0; x < 2; ++x)
          if (((ls.steps[t] >> (12 + 2 * x)) & 3u) == 0u) mbar_arrive(&bar_kempty[s]);
        *reinterpret_cast<volatile int*>(&k_issued) = t + 1;
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------------------------------ V producer (own ring:
    // V is consumed ~2 steps after K, so its stages are requested later and held shorter)
    if (elect_one()) {
      tma_prefetch_desc(&tmV);
      const uint64_t pol_kv = policy_evict_last();
      const int kvrow0 = (gr.b * a.H_kv + kvh) * a.L;
      for (int t = 0; t < T; ++t) {
        const int j = int(ls.steps[t] & 0xFFFu);
        const int s = t % kSV;
        if (t >= kSV) mbar_wait(&bar_vempty[s], ((t / kSV) + 1) & 1);
        mbar_arrive_expect_tx(&bar_vfull[s], SL::kTileBytes);
        tma_load_3d_hint(smem + SL::kVRing + s * SL::kTileBytes, &tmV, &bar_vfull[s], 0, kvrow0 + j * kBS, 0,
                         pol_kv);
        for (int x = 0; x < 2; ++x)
          if (((ls.steps[t] >> (12 + 2 * x)) & 3u) == 0u) mbar_arrive(&bar_vempty[s]);
        *reinterpret_cast<volatile int*>(&v_issued) = t + 1;
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == 3) {
    // ------------------------------------------------------------ MMA issuers
    const int x = warp == 1 ? 0 : 1;
    constexpr uint32_t idesc_s = idesc_f16(128, kBS, /*bf16*/ 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(128, D, /*bf16*/ 1, false, /*V MN-major*/ true);
    const uint32_t tb = tmem + x * 256;
    const uint32_t sQ = smem_u32(smem + x * SL::kQTile);
    const int n_own = ls.n_own[x];
    // union positions of own steps k_pv + 1 .. k_pv + 2 (the window the issuer looks at)
    int pos[3];
    pos[0] = attn::next_own(ls, x, 0, T);
    pos[1] = attn::next_own(ls, x, pos[0] + 1, T);
    // Parity waits are only meaningful within one phase of a barrier. This tile's own
    // positions can be far apart while the stage's barriers advance on positions it skips,
    // so it waits on the full barrier of position p only once the producer has ISSUED load p:
    // that implies load p - kS has landed (the producer waited for its release), i.e. the
    // barrier is at most one phase behind; it cannot be ahead (this tile still holds p).
    auto wait_loaded = [&](uint64_t* full, const int* issued, int p, int nst) {
      while (*reinterpret_cast<const volatile int*>(issued) <= p) __nanosleep(32);
      mbar_wait(&full[p % nst], (p / nst) & 1);
    };
    auto issue_s = [&](int tt, int kk) {  // S(kk) from union position tt into buffer kk & 1
      wait_loaded(bar_kfull, &k_issued, tt, kSK);
      TPTRACE((threadIdx.x & 31) == 0, x, kk, 12);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + SL::kKRing + (tt % kSK) * SL::kTileBytes);
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad = sdesc_sw128(sQ + kc * 128 * 128 + ks * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sK + kc * kBS * 128 + ks * 32, 16, 1024);
            umma_f16_ss(tb + (kk & 1) * 64, ad, bd, idesc_s, (kc | ks) != 0);
          }
        umma_commit(&bar_kempty[tt % kSK]);
        umma_commit(&bar_sfull[x][kk & 1]);
        TPTRACE(true, x, kk, 0);
      }
      __syncwarp();
    };
    mbar_wait(&bar_q[x], 0);  // Q of tile x has landed
    tc_fence_after();
    int ns = 0;  // next own step whose S is not issued yet
    // S(ns) may go once its logit buffer is free: P.V(ns - 2) issued (ns <= k_pv + 2). Ahead of
    // P.V(ns - 1) only if its position lies within kSK union positions of the oldest own step
    // whose P.V is not issued (pos[0]). Deadlock freedom: skipped positions never block (the
    // producers release them), so a tile waits only on the other tile's own uses — S frontier
    // s, P.V frontier f. Waiting on K(s_x) needs s_y > s_x - kSK, on V(f_x) needs f_y > f_x - kSV;
    // a cycle x on K / y on V would need s_x > f_x + kSV + kSK, which this rule excludes (and
    // K/K, V/V cycles contradict themselves).
    auto issue_ready = [&](int k_pv) {
      while (ns < n_own && ns <= k_pv + 2) {
        const int tn = pos[ns - (k_pv + 1)];
        if (ns > k_pv + 1 && tn - pos[0] >= kSK) break;
        issue_s(tn, ns);
        ++ns;
      }
    };
    issue_ready(-1);
    for (int k = 0; k < n_own; ++k) {
      mbar_wait(&bar_pfull[x][k & 1], (k >> 1) & 1);  // P(k) of all 128 rows is in TMEM
      TPTRACE((threadIdx.x & 31) == 0, x, k, 6);
      tc_fence_after();
      const int t = pos[0];
      wait_loaded(bar_vfull, &v_issued, t, kSV);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sV = smem_u32(smem + SL::kVRing + (t % kSV) * SL::kTileBytes);
#pragma unroll
        for (int ks = 0; ks < kBS / 16; ++ks) {
          // keys [16 ks, 16 ks + 16): half ks / 2 stored its P at column 32 * (ks / 2)
          const uint32_t pa = tb + (k & 1) * 64 + (ks >> 1) * 32 + (ks & 1) * 8;
          const uint64_t bd = sdesc_sw128(sV + ks * 16 * 128, kBS * 128, 1024);
          umma_f16_ts(tb + kTO, pa, bd, idesc_o, (k > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(&bar_vempty[t % kSV]);
        umma_commit(&bar_pvdone[x]);
        TPTRACE(true, x, k, 7);
      }
      __syncwarp();
      pos[0] = pos[1];
      pos[1] = attn::next_own(ls, x, pos[0] < T ? pos[0] + 1 : T, T);
      issue_ready(k);
    }
    if (elect_one()) umma_commit(&bar_ofull[x]);
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax / epilogue
    const int lane = threadIdx.x & 31;
    const int x = (warp - 4) >> 3;         // tile
    const int hf = ((warp - 4) >> 2) & 1;  // key half (and O column half)
    const int q = warp & 3;                // TMEM lane quarter
    const int row = q * 32 + lane;
    const int slot = 2 * x + (row >> 6), rloc = row & 63;
    const int g = int((ls.perm >> (2 * slot)) & 3u);
    const int ig = gr.i[g], hg = gr.h[g];
    const bool en = gr.en[g];
    const uint32_t bar_id = 1 + x * 4 + q;  // named barrier of the two halves of these rows
    const uint32_t tb = tmem + (uint32_t(q * 32) << 16) + x * 256;
    const float sl2 = a.scale_log2;
    float m_used = -INFINITY, l = 0.f;
    const int n_own = ls.n_own[x];
    const int c_half = hf * 32;  // first key column of this half
    int t = -1;
    for (int kk = 0; kk < n_own; ++kk) {
      t = attn::next_own(ls, x, t + 1, T);
      const uint32_t e = ls.steps[t];
      const int j = int(e & 0xFFFu);
      const bool sel = (e >> (12 + slot)) & 1u;  // warp-uniform (32 rows of one group)
      const uint32_t sb = tb + (kk & 1) * 64 + c_half;  // this half's S / P columns
      mbar_wait(&bar_sfull[x][kk & 1], (kk >> 1) & 1);
      TPTRACE(row == 0, x, kk, hf ? 8 : 1);
      tc_fence_after();
      uint32_t packed[16];
      if (sel) {
        float sv[32];
        {
          uint32_t v[32];
          tmem_ld32(sb, v);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 32; ++c) sv[c] = __uint_as_float(v[c]);
        }
        TPTRACE(row == 0 && hf == 0, x, kk, 2);
        const bool diag = (j == ig) && !a.noncausal;
        if (diag) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c_half + c > rloc) sv[c] = -INFINITY;
        }
        float m8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(fmaxf(sv[u], sv[8 + u]), fmaxf(sv[16 + u], sv[24 + u]));
        const float hm = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        float (*xb)[2] = xch[kk & 1][x];
        xb[row][hf] = hm;
        named_bar_sync(bar_id, 64);
        const float mx = fmaxf(hm, xb[row][hf ^ 1]) * sl2;
        TPTRACE(row == 0, x, kk, hf ? 9 : 3);
        // lazy rescale: both halves of a row take the same decision (same mx)
        const bool need = mx > m_used + 8.f;
        const bool need_o = need && m_used != -INFINITY;
        if (__any_sync(0xffffffffu, need_o)) {
          // O must hold every key before this step: wait for P.V(kk - 1). Warp-collective
          // TMEM ld/st; rows that did not move use f = 1.
          mbar_wait(&bar_pvdone[x], (kk - 1) & 1);
          tc_fence_after();
          const float f = need_o ? ex2_approx(m_used - mx) : 1.f;
#pragma unroll 1
          for (int c0 = 0; c0 < D / 2; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tb + kTO + hf * (D / 2) + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            US_TMEM_ST_X32(tb + kTO + hf * (D / 2) + c0, o);
          }
          l *= f;
        }
        if (need) m_used = mx;
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m_used, -m_used);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        if (!diag) {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
            float2 p;
            if (c >= 32 - kPoly) {
              p = attn::ex2_poly2(xx);
            } else {
              p.x = ex2_approx(xx.x);
              p.y = ex2_approx(xx.y);
            }
            acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
            packed[c >> 1] = pack_bf16(p.x, p.y);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const float2 xx = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nm);
            float2 p;
            p.x = ex2_approx(xx.x);
            p.y = ex2_approx(xx.y);
            acc[(c >> 1) & 3] = __fadd2_rn(acc[(c >> 1) & 3], p);
            packed[c >> 1] = pack_bf16(p.x, p.y);
          }
        }
        const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        l += s2.x + s2.y;
        TPTRACE(row == 0 && hf == 0, x, kk, 4);
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) packed[c] = 0u;
      }
      // P(k) of this half -> TMEM (inside the S columns this warp itself loaded)
      tmem_st16(sb, packed);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[x][kk & 1]);
      TPTRACE(lane == 0 && q == 0, x, kk, hf ? 10 : 5);
      TPTRACE(lane == 0 && q == 3 && hf == 0, x, kk, 11);
    }
    // ---- epilogue: row sum of both halves, this half of the O columns
    xl[x][row][hf] = l;
    named_bar_sync(bar_id, 64);
    const float lt = l + xl[x][row][hf ^ 1];
    mbar_wait(&bar_ofull[x], 0);
    tc_fence_after();
    const bool write = en && lt > 0.f;
    const float inv_l = 1.f / lt;
    __nv_bfloat16* dst =
        a.O + ((long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + rloc) * D + hf * (D / 2);
#pragma unroll 1
    for (int c0 = 0; c0 < D / 2; c0 += 16) {
      uint32_t o[16];
      tmem_ld16(tb + kTO + hf * (D / 2) + c0, o);
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
    if (write && a.lse && hf == 0)
      a.lse[(long long)(gr.b * a.H + hg) * a.L + (long long)ig * kBS + rloc] =
          (m_used + __log2f(lt)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

template <int D>
us_status launch_tp_t(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                      cudaStream_t st) {
  const int smem = TpSmem<D>::kBytes + 1024;  // + alignment slack
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(attn_tp_kernel<D>, smem, attr_done, "attn_tp_kernel smem attribute"); s != US_OK)
    return s;
  attn_tp_kernel<D><<<unsigned(attn::work_items(a)), kThreads, smem, st>>>(tmQ, tmK, tmV, a);
  US_LAUNCH_CHECK("attn_tp_kernel");
  return US_OK;
}

}  // namespace

us_status launch_attention_tp(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                              const CUtensorMap& tmV, cudaStream_t st) {
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_tp_t<128>(a, tmQ, tmK, tmV, st);
  if (a.D == 64) return launch_tp_t<64>(a, tmQ, tmK, tmV, st);
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us

#if US_TP_TRACE
extern "C" int us_debug_tp_trace(int cta, long long* host_out) {
  if (host_out) return int(cudaMemcpyFromSymbol(host_out, ::g_tp_trace, sizeof(long long) * 2 * 4096 * 16));
  return int(cudaMemcpyToSymbol(::g_tp_trace_cta, &cta, sizeof(int)));
}
#endif
