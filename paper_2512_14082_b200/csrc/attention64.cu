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
// * K/V tiles of 64 keys arrive by TMA in step-major order (round k: the k-th selected block
//   of chain 0, 1, 2, 3) into a K ring and a V ring shared by the four chains, so the rings
//   hold the next steps of every chain (see the producers); four producer warps issue the
//   copies, as one issuing warp caps at ~20-29 B/clk (tools/tma_probe.cu).
// * The four chains' causal mask rows live in shared memory (the producers' walk); all
//   shared memory is dynamic (the rows' size follows W).
// * Q arrives by TMA too: each producer copies one group's 64 rows into a V stage that is
//   idle at CTA start, and the softmax warps move it to TMEM, after which the V stream
//   starts. The softmax warps' own 16-B row loads took ~7 k cycles at CTA start and held
//   the first K copy behind them (a CTA's fixed cost: ~25 k -> ~20 k cycles).
//
// Warps (768 threads): 0 row loader + K producer, 21 K producer, 22-23 V producers, 1-3 and 20
// MMA issuers of groups 0-3 (warp 1 owns TMEM), 4-19 softmax (warp 4 + 4 g + q: group g, lane
// quarter q).
#include "attn_common.cuh"
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

#ifndef US_ATTN_TRACE
#define US_ATTN_TRACE 0
#endif
#if US_ATTN_TRACE
// clock64 step timeline of one CTA (tools/a64_trace.py): [group][own step][event]; event 7 of a
// group step = its load index (a value, not a time); [4][load][0 / 1] = K / V load issued
__device__ long long g_a64_trace[5 * 4096 * 8];  // [group 0-3 | 4 = producer]
__device__ int g_a64_trace_cta = -1;
#define A64_STAMP(g, k, e) \
  do { if (traced && (k) < 4096) g_a64_trace[(((g) * 4096) + (k)) * 8 + (e)] = clock64(); } while (0)
#else
#define A64_STAMP(g, k, e) do { } while (0)
#endif

// ring split (stages of 16 KB at d = 128; twice as many 8 KB stages at d = 64) and the
// number of the four producer warps that issue K (the rest issue V). Measured at C3
// (profiles/r02d): K6/V6 with 2 + 2 producers 5.3-5.5 ms at 64K gain 9; K8/V4 5.5-5.6,
// K7/V5 5.7-5.8, one K producer (3 V) 6.2-7.0.
#ifndef US_A64_KS
#define US_A64_KS 6
#endif
#ifndef US_A64_VS
#define US_A64_VS 6
#endif
#ifndef US_A64_KPROD
#define US_A64_KPROD 2
#endif
// load order: 1 = union (ascending j over the four chains' blocks, a block two chains
// selected loaded once), 0 = step-major (round k: the k-th block of each chain)
#ifndef US_A64_QBY_ISSUER  // 1: group g's MMA issuer warp issues its Q copy at CTA start
#define US_A64_QBY_ISSUER 1  //    (0: the four producers, after the union count, ahead of K / V;
#endif                       //    1 is 40 us faster at 1-32 blocks per row, profiles/r02k)
#ifndef US_A64_UNION
#define US_A64_UNION 1
#endif

namespace us {
namespace {

using attn::kBS;
using attn::kMaxN;

template <int D>
struct A64Smem {
  // K ring: a K tile is held until its S retires; V ring: a V tile until its P.V retires
  static constexpr int kKS = (D == 128 ? 1 : 2) * US_A64_KS;
  static constexpr int kVS = (D == 128 ? 1 : 2) * US_A64_VS;
  static constexpr int kChunks = D / 64;
  static constexpr int kKVBytes = kBS * D * 2;   // one K or V tile of 64 keys
  static constexpr int kRingBytes = (kKS + kVS) * kKVBytes;  // K stages, then V stages
  static constexpr int kPBytes = 64 * kBS * 2;   // per group: 64 rows x 64 keys bf16, SWIZZLE_128B
  // control block (barriers, counters) after the P tiles, then the four mask rows
  struct Ctl {
    uint64_t bar_q[4], bar_kfull[kKS], bar_kempty[kKS], bar_vfull[kVS], bar_vempty[kVS], bar_sfull[4], bar_sfree[4],
        bar_pfull[4], bar_pvdone[4], bar_ofull[4];
    uint64_t bar_qfull[4];  // group g's Q rows have landed in V stage g (TMA)
    uint64_t bar_qfree;     // the 16 softmax warps have read their Q rows: V stages 0-3 are free
    uint32_t tmem_base;
    int k_issued, v_issued;  // loads of the sequence whose K / V the producer has issued
    int n_own[4];            // own steps (selected blocks j <= i) of each chain
  };
  static constexpr int kCtlOff = kRingBytes + 4 * kPBytes;
  static constexpr int kRowsOff = kCtlOff + (int(sizeof(Ctl)) + 15) / 16 * 16;
  // dynamic bytes for W mask words per row; ALL the kernel's shared memory is dynamic (no
  // static __shared__), so the base is the window base, 1024-aligned (checked in the kernel)
  static constexpr int bytes(int W) { return kRowsOff + 16 * W; }
};

constexpr uint32_t kTS = 0, kTO = 64, kTQ = 192;
constexpr int kThreads = 24 * 32;
// columns >= this of each 32-column half of an off-diagonal block: FMA-pipe exp2. 32 = none:
// at C3 the polynomial share only costs (28: +0.5 / +1.3 %, 24: +1.5 / +2.3 %, 16: +4 / +5.5 %
// at gain 9 / 8, profiles/r02d) — the FMA pipe, not the MUFU, is the contended one here
#ifndef US_A64_POLY_FROM
#define US_A64_POLY_FROM 32
#endif
constexpr int kPolyFrom = US_A64_POLY_FROM;

__device__ __forceinline__ int issuer_group(int warp) { return warp == 20 ? 3 : warp - 1; }


template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using SL = A64Smem<D>;
  constexpr int kKS = SL::kKS, kVS = SL::kVS;
  constexpr bool kUnion = US_A64_UNION != 0;
  // union: every chain releases every position (the producer for the chains that skip it);
  // step-major: each load belongs to one chain
  constexpr int kEmptyCount = kUnion ? 4 : 1;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u)) __trap();  // SWIZZLE_128B tiles need 1024-B alignment
  auto& ctl = *reinterpret_cast<typename SL::Ctl*>(smem + SL::kCtlOff);
  auto& bar_q = ctl.bar_q;
  auto& bar_kfull = ctl.bar_kfull;
  auto& bar_kempty = ctl.bar_kempty;
  auto& bar_vfull = ctl.bar_vfull;
  auto& bar_vempty = ctl.bar_vempty;
  auto& bar_sfull = ctl.bar_sfull;
  auto& bar_sfree = ctl.bar_sfree;
  auto& bar_pfull = ctl.bar_pfull;
  auto& bar_pvdone = ctl.bar_pvdone;
  auto& bar_ofull = ctl.bar_ofull;
  auto& k_issued = ctl.k_issued;
  auto& v_issued = ctl.v_issued;
  auto& n_own = ctl.n_own;
  uint32_t* const mrow = reinterpret_cast<uint32_t*>(smem + SL::kRowsOff);  // [4][W]: causal rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if US_ATTN_TRACE
  const bool traced = int(blockIdx.x) == g_a64_trace_cta;
#endif
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
  if (a.sel_pairs && !attn::m64_wins(a, gr.b, kvh)) return;  // dense enough for attn_kernel
  if (threadIdx.x == 0) {
    A64_STAMP(4, 4090, 0);  // (trace) CTA lifecycle: entry
    // the tensor-map descriptors, well before the first copy needs them
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  // mask row of chain g (its selected key blocks; read through L1 by the cursors below)
  auto row_of = [&](int g) {
    return a.mask + ((long long)(gr.b * a.planes + gr.h[g] / a.heads_per_plane) * a.N + gr.i[g]) * a.W;
  };

  if (threadIdx.x == 32) {
    for (int g = 0; g < 4; ++g) {
      mbar_init(&bar_q[g], 4);
      mbar_init(&bar_sfull[g], 1);
      mbar_init(&bar_sfree[g], 4);
      mbar_init(&bar_pfull[g], 4);
      mbar_init(&bar_pvdone[g], 1);
      mbar_init(&bar_ofull[g], 1);
    }
    for (int g = 0; g < 4; ++g) mbar_init(&ctl.bar_qfull[g], 1);
    mbar_init(&ctl.bar_qfree, 16);
    for (int s = 0; s < kKS; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], kEmptyCount);
    }
    for (int s = 0; s < kVS; ++s) {
      mbar_init(&bar_vfull[s], 1);
      mbar_init(&bar_vempty[s], kEmptyCount);
    }
    k_issued = v_issued = 0;
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&ctl.tmem_base, 512);
  if (threadIdx.x == 32) A64_STAMP(4, 4091, 1);  // (trace) TMEM allocated
  if (warp < 4) {
    // warp g: chain g's causal row -> shared memory, its own steps (popcount) and the
    // asynchronous data-error report (the reference throws, attention.cpp:106-108,
    // 127-129): a non-causal bit anywhere in the row, or an empty causal prefix
    const int g = warp;
    unsigned c = 0, bad = 0;
    const uint32_t* src = row_of(g);
    const int ig = gr.i[g];
    for (int w = lane; w < a.W; w += 32) {
      const uint32_t word = gr.en[g] ? src[w] : 0u;
      const int lo = w << 5;
      const uint32_t keep = lo > ig ? 0u : (ig - lo >= 31 ? ~0u : (2u << (ig - lo)) - 1u);
      bad |= word & ~keep;
      c += __popc(word & keep);
      mrow[g * a.W + w] = word & keep;
    }
    c = __reduce_add_sync(0xffffffffu, c);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
      n_own[g] = int(c);
      if (a.err && gr.en[g] && (bad || c == 0)) {
        atomicOr(a.err, bad ? 4u : 8u);
        atomicMin(a.first_bad, int32_t((src - a.mask) / a.W));
      }
    }
    if (threadIdx.x == 0) A64_STAMP(4, 4091, 0);  // (trace) row 0 in shared memory
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) A64_STAMP(4, 4090, 1);  // (trace) prologue barrier passed
  const uint32_t tmem = ctl.tmem_base;
  const int n0 = n_own[0], n1 = n_own[1], n2 = n_own[2], n3 = n_own[3];
  // index of chain g's own step k in the load sequence (round k: chains 0-3 in order, a
  // chain with fewer than k + 1 steps skipped)
  auto seq_index = [&](int g, int k) {
    return min(k, n0) + min(k, n1) + min(k, n2) + min(k, n3) + (g > 0 && n0 > k) + (g > 1 && n1 > k) +
           (g > 2 && n2 > k);
  };
  auto union_count = [&]() {  // (warp-wide) blocks any chain selected
    unsigned nu = 0;
    for (int w = lane; w < a.W; w += 32)
      nu += __popc(mrow[w] | mrow[a.W + w] | mrow[2 * a.W + w] | mrow[3 * a.W + w]);
    return int(__reduce_add_sync(0xffffffffu, nu));
  };
  auto union_word = [&](int w) {
    return mrow[w] | mrow[a.W + w] | mrow[2 * a.W + w] | mrow[3 * a.W + w];
  };
  // union mode: chain g's own positions in ascending order, as union indices
  struct OwnWalk {
    int w = 0, base = 0;
    uint32_t own = 0u, uni = 0u;
  };
  auto own_start = [&](int g) {
    OwnWalk x;
    x.own = mrow[g * a.W];
    x.uni = union_word(0);
    return x;
  };
  auto own_next = [&](OwnWalk& x, int g) {
    while (x.own == 0u) {
      x.base += __popc(x.uni);
      ++x.w;
      x.own = mrow[g * a.W + x.w];
      x.uni = union_word(x.w);
    }
    const int b = __ffs(x.own) - 1;
    x.own &= x.own - 1u;
    return x.base + __popc(x.uni & ((1u << b) - 1u));
  };

  if (warp == 0 || warp >= 21) {
    // ------------------------------------------------------------ TMA producers
    // The load sequence (US_A64_UNION): union order — ascending j over the four chains'
    // selected blocks, a block several chains selected loaded once (0.74 / 0.56 loads per
    // own step at C3 gain 9 / 8), the producer releasing each position for the chains that
    // skip it — or step-major (round k = the k-th block of chain 0, 1, 2, 3; every load
    // belongs to one chain). K and V are two sequences (a K tile is only held until its S
    // retires, so K runs ahead): K(u) once K stage u % kKS is free, V(u) once V stage
    // u % kVS is. One warp issues only ~20-29 B/clk of bulk / tensor copies however deep
    // its ring (tools/tma_probe.cu: the copies of one issuing warp proceed one at a time;
    // four issuing warps reach the ~70 B/clk/SM L2 -> SMEM ceiling), so each sequence is
    // dealt round-robin to two warps (K: warps 0, 21; V: warps 22, 23). Arming a load
    // (stage free, expect_tx, skip releases, the issued count) stays in sequence order;
    // the copies run in parallel.
    const int pw = warp == 0 ? 0 : warp - 20;  // 0 .. kKProd - 1: K producers; the rest V
    constexpr int kKProd = US_A64_KPROD;
    const bool is_v = pw >= kKProd;
    const int np = is_v ? 4 - kKProd : kKProd, me = is_v ? pw - kKProd : pw;
    const int total = kUnion ? union_count() : n0 + n1 + n2 + n3;  // loads of the sequence
    if (threadIdx.x == 0) A64_STAMP(4, 4091, 3);  // (trace) producer 0: union counted
    if (elect_one()) {
      // first, producer pw's copy of group pw's 64 Q rows (16 KB at d = 128) into V stage pw,
      // idle until the first V loads: four producers issue them at once (one issuing warp's
      // copies proceed one at a time), fully coalesced — the softmax warps' own 16-B row
      // loads of Q took ~7 k cycles at CTA start and held the first K copy behind them
      if (!US_A64_QBY_ISSUER) {
        const int gq = pw;
        if (gr.en[gq]) {
          mbar_arrive_expect_tx(&ctl.bar_qfull[gq], SL::kKVBytes);
          tma_load_3d_hint(smem + (kKS + gq) * SL::kKVBytes, &tmQ, &ctl.bar_qfull[gq], 0,
                           (gr.b * a.H + gr.h[gq]) * a.L + gr.i[gq] * kBS, 0, policy_evict_first());
        } else {
          mbar_arrive(&ctl.bar_qfull[gq]);
        }
      }
      if (is_v) mbar_wait(&ctl.bar_qfree, 0);  // V stages 0-3 hold Q until the softmax warps read it
      const uint64_t pol_kv = policy_evict_last();
      const int kvrow0 = (gr.b * a.H_kv + kvh) * a.L;
      const int nmax = max(max(n0, n1), max(n2, n3));
      const CUtensorMap* tm = is_v ? &tmV : &tmK;
      const int nst = is_v ? kVS : kKS;
      uint64_t* full = is_v ? bar_vfull : bar_kfull;
      uint64_t* empty = is_v ? bar_vempty : bar_kempty;
      int* issued = is_v ? &v_issued : &k_issued;
      uint8_t* ring = smem + (is_v ? kKS : 0) * SL::kKVBytes;
      // walk of the sequence: step-major (round k, chain g) with a bit cursor per chain, or
      // the union bits (word uw, remaining bits ub)
      int k = 0, g = 0, w[4] = {0, 0, 0, 0};
      uint32_t bits[4];
      for (int c = 0; c < 4; ++c) bits[c] = mrow[c * a.W];
      int uw = 0;
      uint32_t ub = union_word(0);
      for (int u = 0; u < total; ++u) {
        int j;
        if (kUnion) {
          while (ub == 0u) ub = union_word(++uw);
          j = (uw << 5) + __ffs(ub) - 1;
          ub &= ub - 1u;
        } else {
          while (k < nmax && k >= n_own[g]) {
            if (++g == 4) { g = 0; ++k; }
          }
          while (bits[g] == 0u) bits[g] = mrow[g * a.W + ++w[g]];
          j = (w[g] << 5) + __ffs(bits[g]) - 1;
          bits[g] &= bits[g] - 1u;
          if (++g == 4) { g = 0; ++k; }
        }
        if (u % np != me) continue;  // another producer's load of this sequence
        const int s = u % nst;
        while (ld_acquire_cta(issued) < u) {
        }
        // (load u - nst armed => load u - 2 nst released: the parity wait is within one phase)
        if (u >= nst) mbar_wait(&empty[s], ((u / nst) + 1) & 1);
        mbar_arrive_expect_tx(&full[s], SL::kKVBytes);
        if (kUnion) {
          // a chain whose group skips this position releases it right away (the producer
          // arrives for it): a chain only ever holds the stages of its own positions
          const int wj = j >> 5;
          const uint32_t bj = 1u << (j & 31);
          for (int c = 0; c < 4; ++c)
            if ((mrow[c * a.W + wj] & bj) == 0u) mbar_arrive(&empty[s]);
        }
        st_release_cta(issued, u + 1);
        tma_load_3d_hint(ring + s * SL::kKVBytes, tm, &full[s], 0, kvrow0 + j * kBS, 0, pol_kv);
        A64_STAMP(4, u, is_v ? 1 : 0);  // (trace) K / V load u issued
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
    const int n = n_own[g];
    // K (V) of load u: a parity wait is only meaningful within one phase of the barrier, so
    // the chain waits on kfull(u) only once the producer has ISSUED load u — which implies
    // load u - kKS has landed (its release needed it); the barrier cannot be ahead (this
    // chain holds u).
    auto wait_k = [&](int u) {
      while (ld_acquire_cta(&k_issued) <= u) __nanosleep(20);
      mbar_wait(&bar_kfull[u % kKS], (u / kKS) & 1);
    };
    auto wait_v = [&](int u) {
      while (ld_acquire_cta(&v_issued) <= u) __nanosleep(20);
      mbar_wait(&bar_vfull[u % kVS], (u / kVS) & 1);
    };
    auto issue_s = [&](int kk, int u) {
      A64_STAMP(g, kk, 3);  // S(kk) wants to issue
      wait_k(u);
      A64_STAMP(g, kk, 4);  // ... its K landed: issued
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + (u % kKS) * SL::kKVBytes);
#pragma unroll
        for (int kc = 0; kc < SL::kChunks; ++kc)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc_sw128(sK + kc * kBS * 128 + ks * 32, 16, 1024);
            umma_f16_ts(tb + kTS, tb + kTQ + (kc * 4 + ks) * 8, bd, idesc_s, (kc | ks) != 0);
          }
        umma_commit(&bar_sfull[g]);
        umma_commit(&bar_kempty[u % kKS]);
      }
      __syncwarp();
    };
    if (US_A64_QBY_ISSUER) {
      // group g's 64 Q rows (16 KB at d = 128) into V stage g; this warp is idle until they
      // are in TMEM, and the producers' first copies are then K / V only
      if (elect_one()) {
        if (gr.en[g]) {
          mbar_arrive_expect_tx(&ctl.bar_qfull[g], SL::kKVBytes);
          tma_load_3d_hint(smem + (kKS + g) * SL::kKVBytes, &tmQ, &ctl.bar_qfull[g], 0,
                           (gr.b * a.H + gr.h[g]) * a.L + gr.i[g] * kBS, 0, policy_evict_first());
        } else {
          mbar_arrive(&ctl.bar_qfull[g]);
        }
      }
      __syncwarp();
    }
    mbar_wait(&bar_q[g], 0);  // Q rows of group g are in TMEM
    tc_fence_after();
    OwnWalk ow = own_start(g);
    int u_next = n > 0 ? (kUnion ? own_next(ow, g) : seq_index(g, 0)) : -1;  // load index of own step k
    if (n > 0) issue_s(0, u_next);
    for (int k = 0; k < n; ++k) {
      const int u = u_next;
      const int u1 = k + 1 < n ? (kUnion ? own_next(ow, g) : seq_index(g, k + 1)) : -1;
      u_next = u1;
      // S(k+1) right after the softmax has loaded S(k) when its K has landed (a non-blocking
      // probe: P.V(k) is not held up by a late K), otherwise after P.V(k). Step-major order
      // could also block here (K(u) needs only the S MMAs of earlier loads); in union order
      // a blocking wait is only safe within kKS positions of u: the stage then last held a
      // position before u, which every chain releases without waiting on this one.
      mbar_wait(&bar_sfree[g], k & 1);
      const bool early =
          u1 >= 0 && ((kUnion && u1 - u < kKS) || (ld_acquire_cta(&k_issued) > u1 &&
                                                   mbar_test_wait(&bar_kfull[u1 % kKS], (u1 / kKS) & 1)));
      if (early) issue_s(k + 1, u1);
      mbar_wait(&bar_pfull[g], k & 1);  // P(k) of the group's 64 rows is in SMEM
      wait_v(u);
      A64_STAMP(g, k, 5);  // P(k) seen and V landed: P.V(k) issued
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sV = smem_u32(smem + (kKS + u % kVS) * SL::kKVBytes);
#pragma unroll
        for (int ks = 0; ks < kBS / 16; ++ks) {
          const uint64_t ad = sdesc_sw128(sP + ks * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sV + ks * 16 * 128, kBS * 128, 1024);
          umma_f16_ss(tb + kTO, ad, bd, idesc_o, (k > 0 || ks > 0) ? 1u : 0u);
        }
        umma_commit(&bar_vempty[u % kVS]);
        umma_commit(&bar_pvdone[g]);
      }
      __syncwarp();
      if (!early && u1 >= 0) issue_s(k + 1, u1);
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
      // this half of the Q row: from V stage g (the producers' SWIZZLE_128B copy: d-chunk c of
      // row r at c * 8 KB + r * 128, 16-B unit u at (u ^ (r & 7)) * 16) -> TMEM (A operand of
      // S = Q K^T, 2 bf16 per column)
      constexpr int kQv = D / 16;  // 16-B units per half row
      uint4 qv[kQv];
      mbar_wait(&ctl.bar_qfull[g], 0);
      const uint8_t* qs = smem + (kKS + g) * SL::kKVBytes;
#pragma unroll
      for (int u = 0; u < kQv; ++u) {
        const int U = half * kQv + u, c = U >> 3, cu = U & 7;
        qv[u] = en ? *reinterpret_cast<const uint4*>(qs + c * 8192 + r * 128 + ((cu ^ (r & 7)) << 4))
                   : make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ctl.bar_qfree);  // (release: the reads above are done)
#pragma unroll
      for (int c0 = 0; c0 < D / 4; c0 += 16) {
        uint32_t w16[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 v = qv[c0 / 4 + u];
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
      if (threadIdx.x == 128) A64_STAMP(4, 4090, 2);  // (trace) chain 0 quarter 0: Q in TMEM
    }
    const int n = n_own[g];
    // own blocks ascend and end at j <= i: only the last can be the diagonal block
    const bool diag_sel = n > 0 && ((mrow[g * a.W + (ig >> 5)] >> (ig & 31)) & 1u);
    for (int k = 0; k < n; ++k) {
      if (threadIdx.x % 128 == 0) A64_STAMP(g, k, 0);  // softmax (quarter 0) wants S(k)
#if US_ATTN_TRACE
      if (traced && threadIdx.x % 128 == 0 && k < 4096) g_a64_trace[((g * 4096) + k) * 8 + 7] = seq_index(g, k);
#endif
      mbar_wait(&bar_sfull[g], k & 1);
      if (threadIdx.x % 128 == 0) A64_STAMP(g, k, 1);  // S(k) seen
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
      const bool diag = diag_sel && k == n - 1;
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
      if (threadIdx.x % 128 == 0) A64_STAMP(g, k, 2);  // exponentials done
      if (!pv_prev_done) mbar_wait(&bar_pvdone[g], (k - 1) & 1);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        st_shared_v4(prow + (((4 * half + c) ^ (r & 7)) << 4), packed[4 * c], packed[4 * c + 1], packed[4 * c + 2],
                     packed[4 * c + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_pfull[g]);
      if (threadIdx.x % 128 == 0) A64_STAMP(g, k, 6);  // P(k) handed off
    }
    // ---- epilogue: the row sum of both halves, this half of the O columns
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    mbar_wait(&bar_ofull[g], 0);
    if (threadIdx.x == 128) A64_STAMP(4, 4090, 3);  // (trace) O complete
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
  if (threadIdx.x == 128) A64_STAMP(4, 4090, 4);  // (trace) chain 0 quarter 0: epilogue stored
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 32) A64_STAMP(4, 4090, 5);  // (trace) TMEM released: exit
}

// Selected key blocks j <= i of every mask row (one warp per row, lanes over the row's
// words), and their total over the heads (a.sel_pairs, the density gate's input).
__global__ void __launch_bounds__(256) attn64_counts_kernel(AttnArgs a) {
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
    if (lane == 0) {
      a.row_counts[r] = int32_t(n);
      if (a.sel_pairs && n) {  // per (b, KV head) of each head the plane's row stands for
        const int G = a.H / a.H_kv;
        const int b = int(r / ((long long)a.planes * a.N)), pl = int((r / a.N) % a.planes);
        for (int h = pl * a.heads_per_plane; h < (pl + 1) * a.heads_per_plane; ++h)
          atomicAdd(&a.sel_pairs[b * a.H_kv + h / G], (unsigned long long)n);
      }
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
us_status launch_a64_t(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                       cudaStream_t st) {
  static_assert(A64Smem<D>::bytes(attn::kMaxW) <= 227 * 1024, "attn64_kernel shared memory");
  const int smem = A64Smem<D>::bytes(a.W);
  static std::atomic<uint64_t> attr_done{0};  // (the attribute: the largest W)
  if (us_status s = ensure_smem_attr(attn64_kernel<D>, A64Smem<D>::bytes(attn::kMaxW), attr_done,
                                     "attn64_kernel smem attribute");
      s != US_OK)
    return s;
  long long items = attn::work_items(a);
  if (a.items) {
    if (a.sel_pairs)
      US_CUDA_TRY(cudaMemsetAsync(a.sel_pairs, 0, sizeof(unsigned long long) * a.B * a.H_kv, st), "sel_pairs reset");
    const long long rows = (long long)a.B * a.planes * a.N;
    attn64_counts_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(a);
    US_LAUNCH_CHECK("attn64_counts_kernel");
    attn64_items_kernel<<<unsigned(a.B * a.H_kv), 1024, (a.N + 2) * 4, st>>>(a);
    US_LAUNCH_CHECK("attn64_items_kernel");
    items = (long long)a.B * a.H_kv * ((a.H / a.H_kv * a.N + 3) / 4);
  }
  attn64_kernel<D><<<unsigned(items), kThreads, smem, st>>>(tmQ, tmK, tmV, a);
  US_LAUNCH_CHECK("attn64_kernel");
  return US_OK;
}

}  // namespace

long long attention64_item_entries(int B, int H, int H_kv, int N) {
  return (long long)B * H_kv * ((H / H_kv * N + 3) / 4) * 4;
}

size_t attention64_ws_bytes(int B, int H, int H_kv, int N) {
  return 4 * size_t(attention64_item_entries(B, H, H_kv, N)) + 8 * size_t(B) * H_kv + 4 * size_t(B) * H * N;
}

us_status launch_attention64(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                             cudaStream_t st) {
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  if (a.D == 128) return launch_a64_t<128>(a, tmQ, tmK, tmV, st);
  if (a.D == 64) return launch_a64_t<64>(a, tmQ, tmK, tmV, st);
  set_error("attention: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us

#if US_ATTN_TRACE
extern "C" int us_debug_a64_trace(int cta, long long* host_out) {
  if (host_out) return int(cudaMemcpyFromSymbol(host_out, ::g_a64_trace, sizeof(long long) * 5 * 4096 * 8));
  return int(cudaMemcpyToSymbol(::g_a64_trace_cta, &cta, sizeof(int)));
}
#endif
