// attention_kt.cu — block-sparse FlashAttention forward with KEYS as the MMA M
// dimension (block_sparse_attention, attention.cpp:89-137).
//
// Why transposed. A query block is 64 rows; a UMMA tile is M = 128 rows (M = 64
// issues at the same cost). With queries as M, one tile must hold two query
// groups whose selections are independent, so every step runs the UNION of two
// selections — 47 % of the issued rows were P = 0 at C3 (attention.cu). Here a
// work item is ONE query group (head h, query block i) and M = 128 is a PAIR of
// its own selected key blocks (j_a, j_b, consecutive in ascending order):
//   S^T[128 keys][64 queries] = K_pair . Q^T           (SS, A = K K-major, B = Q K-major)
//   O^T[d=128][64 queries]   += V_pair^T . P^T          (SS, A = V MN-major, B = P^T MN-major)
// so every issued MMA row is a selected (key, query) pair; an odd count wastes
// half of one step per item. Measured issue cost (tools/mma_pattern.py, B200):
// 768 cycles per pair step = 384 per selected 64x64 block, vs 524 per M=128
// tile step of attention.cu (~490 per selected block at 53 % useful rows).
//
// Softmax in the transposed layout: thread = key (TMEM lane), columns = queries.
// The per-query running max would need a cross-lane reduction every step, so the
// offsets m[q] are only moved when some logit exceeds m[q] + kT (log2 units):
// each step ONE barrier-OR vote over the softmax threads decides whether this
// step needs a (rare) exact column-max reduction + rescale of O^T and of the
// per-thread row-sum partials l[q]. The first step of an item always reduces
// (m starts at the first pair's exact column max). Values p = 2^(x - m) <= 2^kT
// are far inside the bf16 / fp32 range; exponent underflow below 2^-126 of the
// running max is the same flush as any FlashAttention kernel. The row sums stay
// as per-thread partials (one per query column) and are reduced once per item.
//
// Roles (32 * (4 + 4*NCG) threads, one CTA per SM, persistent over items):
//   warp 0  item scheduler (static round-robin over a KV-head-major, heaviest-
//           first order) + Q / K TMA producer
//   warp 1  TMEM owner + MMA issuer (one elected lane): S(g+2) is issued right
//           after P.V(g), so the next logits are ready when the softmax needs them
//   warp 2  V TMA producer (own ring: V is consumed ~1 step after K)
//   warps 4 .. 4+4*NCG-1  softmax + epilogue; warp % 4 = TMEM lane quarter,
//           (warp - 4) / 4 = which 64/NCG query columns it owns
// TMEM (512 cols): S^T buffers [0,64) [64,128), O^T buffers [128,192) [192,256).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

#include <cstdlib>

// Debug timeline (tools/kt_trace.py, build with -DUS_KT_TRACE=1): clock64 stamps per
// pair step g < 4096 of the traced CTA (event ids listed in tools/kt_trace.py).
#ifndef US_KT_TRACE
#define US_KT_TRACE 0
#endif
#if US_KT_TRACE
__device__ long long g_kt_trace[4096 * 16];
__device__ int g_kt_trace_cta;
#define KTR(g, e)                                                                    \
  do {                                                                               \
    if (kt_traced && (g) < 4096) g_kt_trace[(long long)(g) * 16 + (e)] = clock64(); \
  } while (0)
#else
#define KTR(g, e) \
  do {            \
  } while (0)
#endif

namespace us {
namespace {

constexpr int kBS = 64;
constexpr int kMaxN = 4096;
constexpr int kMaxW = kMaxN / 32;
#ifndef US_KT_KST
#define US_KT_KST 3
#endif
#ifndef US_KT_QST
#define US_KT_QST 1
#endif
constexpr int kKST = US_KT_KST;  // K pair stages (32 KB each)
constexpr int kVST = 2;   // V pair stages (32 KB each)
constexpr int kQST = US_KT_QST;  // Q tiles (16 KB each)
constexpr int kIR = 4;    // item ring depth
constexpr float kT = 16.f;  // rescale threshold (log2 units)

struct KtSmem {
  static constexpr int kPair = 2 * kBS * 128 * 2;  // 128 rows x 128 d bf16 = 32 KB
  static constexpr int kK = 0;
  static constexpr int kV = kK + kKST * kPair;
  static constexpr int kQ = kV + kVST * kPair;
  static constexpr int kP = kQ + kQST * kBS * 128 * 2;
  static constexpr int kBytes = kP + 2 * 128 * 128;  // P^T x 2: 128 key rows x 128 B
};

struct KtItem {
  int b, h, i, n;       // batch, head, query block, selected blocks (0: empty row)
  int diag;             // the diagonal block i is selected (it is the last one)
  int row;              // mask row index ((b*planes + plane)*N + i)
  uint32_t bits[kMaxW]; // mask row restricted to j <= i
};

__device__ __forceinline__ void decode_kt(const AttnArgs& a, long long item, int& b, int& h, int& i) {
  // (b, kv head) outermost, then query blocks heaviest first, then the G heads
  const int G = a.H / a.H_kv;
  const long long per_kv = (long long)a.N * G;
  const long long bk = item / per_kv;
  const int r = int(item - bk * per_kv);
  i = a.N - 1 - r / G;
  b = int(bk / a.H_kv);
  h = int(bk % a.H_kv) * G + r % G;
}

template <int NCG>
__global__ void __launch_bounds__(32 * (4 + 4 * NCG), 1)
    attn_kt_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  constexpr int CPT = 64 / NCG;       // query columns per softmax thread
  constexpr int NSM = 4 * NCG;        // softmax warps
  constexpr uint32_t kSmThreads = 32 * NSM;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_kfull[kKST], bar_kempty[kKST], bar_vfull[kVST], bar_vempty[kVST], bar_qfull[kQST],
      bar_qempty[kQST], bar_sfull[2], bar_sfree[2], bar_pfull[2], bar_pempty[2], bar_ofull[2], bar_oempty[2],
      bar_ifull[kIR], bar_iempty[kIR];
  __shared__ uint32_t tmem_base_sh;
  __shared__ KtItem items[kIR];
  __shared__ float red[4][64];   // per lane quarter column reductions
  __shared__ float colv[64];     // reduced per-column values

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n_items = (long long)a.B * a.H * a.N;
#if US_KT_TRACE
  const bool kt_traced = int(blockIdx.x) == g_kt_trace_cta;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKST; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], 1);
    }
    for (int s = 0; s < kVST; ++s) {
      mbar_init(&bar_vfull[s], 1);
      mbar_init(&bar_vempty[s], 1);
    }
    for (int s = 0; s < kQST; ++s) {
      mbar_init(&bar_qfull[s], 1);
      mbar_init(&bar_qempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sfree[s], NSM);
      mbar_init(&bar_ofull[s], 1);
      mbar_init(&bar_oempty[s], NSM);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_pfull[s], NSM);
      mbar_init(&bar_pempty[s], 1);
    }
    for (int s = 0; s < kIR; ++s) {
      mbar_init(&bar_ifull[s], 1);
      mbar_init(&bar_iempty[s], 2 + NSM);  // MMA warp, V producer, softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int G = a.H / a.H_kv;

  if (warp == 0) {
    // ------------------------------------------------------------ scheduler + Q/K producer
    // Every item put in the ring has at least one selected block; an empty row (the
    // reference throws, attention.cpp:106-108) is flagged in a.err and written here as
    // O = 0, lse = -inf without entering the pipeline.
    const uint64_t pol = policy_evict_last(), pol_q = policy_evict_first();  // K/V reused, Q streamed
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
    }
    int it = 0, qi = 0;
    long long g = 0;  // global pair step (lane 0)
    for (long long item = blockIdx.x;; item += gridDim.x) {
      const int slot = it % kIR;
      if (it >= kIR) mbar_wait(&bar_iempty[slot], ((it / kIR) + 1) & 1);
      KtItem& I = items[slot];
      if (item >= n_items) {
        if (lane == 0) {
          I.n = -1;  // end of stream
          mbar_arrive(&bar_ifull[slot]);
        }
        break;
      }
      int b, h, i;
      decode_kt(a, item, b, h, i);
      const int row = (b * a.planes + h / a.heads_per_plane) * a.N + i;
      const uint32_t* src = a.mask ? a.mask + (long long)row * a.W : nullptr;
      const int nw = (i >> 5) + 1;
      int cnt = 0;
      uint32_t bad = 0;
      for (int w = lane; w < (src ? a.W : nw); w += 32) {
        uint32_t word = src ? __ldg(src + w) : ~0u;
        uint32_t keep = w < nw ? ~0u : 0u;
        if (w == nw - 1 && (i & 31) < 31) keep = (2u << (i & 31)) - 1u;
        bad |= word & ~keep;
        word &= keep;
        if (w < nw) I.bits[w] = word;
        cnt += __popc(word);
      }
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      bad = __reduce_or_sync(0xffffffffu, bad);
      if (lane == 0 && a.err && (bad || cnt == 0)) {
        atomicOr(a.err, bad ? 4u : 8u);
        atomicMin(a.first_bad, row);
      }
      const long long orow0 = (long long)(b * a.H + h) * a.L + (long long)i * kBS;
      if (cnt == 0) {
        uint4* d4 = reinterpret_cast<uint4*>(a.O + orow0 * 128);
        for (int e = lane; e < kBS * 128 / 8; e += 32) d4[e] = make_uint4(0, 0, 0, 0);
        if (a.lse)
          for (int c = lane; c < kBS; c += 32) a.lse[orow0 + c] = -INFINITY;
        continue;
      }
      __syncwarp();
      if (lane == 0) {
        I.b = b;
        I.h = h;
        I.i = i;
        I.n = cnt;
        I.diag = (I.bits[i >> 5] >> (i & 31)) & 1u;
        I.row = row;
        mbar_arrive(&bar_ifull[slot]);
        // Q tile of the item
        const int qs = qi % kQST;
        if (qi >= kQST) mbar_wait(&bar_qempty[qs], ((qi / kQST) + 1) & 1);
        mbar_arrive_expect_tx(&bar_qfull[qs], kBS * 128 * 2);
        tma_load_3d_hint(smem + KtSmem::kQ + qs * kBS * 256, &tmQ, &bar_qfull[qs], 0, int(orow0), 0, pol_q);
        // K pairs, ascending
        const int kvrow0 = (b * a.H_kv + h / G) * a.L;
        int left = cnt, w = 0;
        uint32_t word = I.bits[0];
        while (left > 0) {
          int j2[2] = {0, 0};
          const int take = left >= 2 ? 2 : 1;
          for (int u = 0; u < take; ++u) {
            while (word == 0u) word = I.bits[++w];
            j2[u] = (w << 5) + __ffs(word) - 1;
            word &= word - 1u;
          }
          const int s = int(g % kKST);
          if (g >= kKST) mbar_wait(&bar_kempty[s], ((g / kKST) + 1) & 1);
          uint8_t* sk = smem + KtSmem::kK + s * KtSmem::kPair;
          mbar_arrive_expect_tx(&bar_kfull[s], take * kBS * 256);
          for (int u = 0; u < take; ++u)
            for (int c = 0; c < 2; ++c)
              tma_load_2d_hint(sk + c * 16384 + u * 8192, &tmK, &bar_kfull[s], c * 64, kvrow0 + j2[u] * kBS, pol);
          KTR(g, 8);
          left -= take;
          ++g;
        }
      }
      __syncwarp();
      ++qi;
      ++it;
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ V producer (lane 0)
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      tma_prefetch_desc(&tmV);
      long long g = 0;
      for (int it = 0;; ++it) {
        const int slot = it % kIR;
        mbar_wait(&bar_ifull[slot], (it / kIR) & 1);
        const KtItem& I = items[slot];
        const int cnt = I.n;
        if (cnt < 0) break;
        const int kvrow0 = (I.b * a.H_kv + I.h / G) * a.L;
        int left = cnt, w = 0;
        uint32_t word = I.bits[0];
        while (left > 0) {
          int j2[2] = {0, 0};
          const int take = left >= 2 ? 2 : 1;
          for (int u = 0; u < take; ++u) {
            while (word == 0u) word = I.bits[++w];
            j2[u] = (w << 5) + __ffs(word) - 1;
            word &= word - 1u;
          }
          const int s = int(g % kVST);
          if (g >= kVST) mbar_wait(&bar_vempty[s], ((g / kVST) + 1) & 1);
          uint8_t* sv = smem + KtSmem::kV + s * KtSmem::kPair;
          mbar_arrive_expect_tx(&bar_vfull[s], take * kBS * 256);
          for (int u = 0; u < take; ++u)
            tma_load_3d_hint(sv + u * 16384, &tmV, &bar_vfull[s], 0, kvrow0 + j2[u] * kBS, 0, pol);
          KTR(g, 9);
          left -= take;
          ++g;
        }
        mbar_arrive(&bar_iempty[slot]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Two cursors over the same pair-step stream: S runs two steps ahead of P.V.
    // Every ring item is non-empty, so the S cursor is at most two items ahead of
    // the P.V cursor (the ring holds four).
    constexpr uint32_t idesc_s = idesc_f16(128, 64, 1, false, false);
    constexpr uint32_t idesc_o = idesc_f16(128, 64, 1, true, true);
    const uint32_t sP = smem_u32(smem + KtSmem::kP);
    struct Cur {
      int it, t, np, n, qi, oi;
      long long g;
    };
    auto fetch = [&](Cur& c) -> bool {
      const int slot = c.it % kIR;
      mbar_wait(&bar_ifull[slot], (c.it / kIR) & 1);
      const int n = items[slot].n;
      if (n < 0) return false;
      c.n = n;
      c.np = (n + 1) / 2;
      c.t = 0;
      return true;
    };
    auto advance = [&](Cur& c, bool& ok, bool release) {
      ++c.g;
      if (++c.t == c.np) {
        if (release) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_iempty[c.it % kIR]);
        }
        ++c.it;
        ++c.qi;
        ++c.oi;
        ok = fetch(c);
      }
    };
    auto issue_s = [&](const Cur& c) {
      const int kst = int(c.g % kKST), sb = int(c.g & 1), qs = c.qi % kQST;
      if (c.t == 0) mbar_wait(&bar_qfull[qs], (c.qi / kQST) & 1);
      mbar_wait(&bar_kfull[kst], (c.g / kKST) & 1);
      if (c.g >= 2) mbar_wait(&bar_sfree[sb], ((c.g >> 1) + 1) & 1);
      tc_fence_after();
      if (lane == 0) KTR(c.g, 10);
      if (elect_one()) {
        const uint32_t sK = smem_u32(smem + KtSmem::kK + kst * KtSmem::kPair);
        const uint32_t sQ = smem_u32(smem + KtSmem::kQ + qs * kBS * 256);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t c2 = uint32_t(kk >> 2), ks = uint32_t(kk & 3) * 32;
          umma_f16_ss(tmem + sb * 64, sdesc_sw128(sK + c2 * 16384 + ks, 16, 1024),
                      sdesc_sw128(sQ + c2 * 8192 + ks, 16, 1024), idesc_s, kk > 0);
        }
        umma_commit(&bar_sfull[sb]);
        umma_commit(&bar_kempty[kst]);
        if (c.t == c.np - 1) umma_commit(&bar_qempty[qs]);
        KTR(c.g, 0);
      }
      __syncwarp();
    };
    Cur cs{0, 0, 0, 0, 0, 0, 0}, cp{0, 0, 0, 0, 0, 0, 0};
    bool s_ok = fetch(cs);
    bool p_ok = fetch(cp);
    for (int k = 0; k < 2 && s_ok; ++k) {  // prologue: S(0), S(1)
      issue_s(cs);
      advance(cs, s_ok, false);
    }
    while (p_ok) {
      // S(g+2) as soon as the softmax has loaded S(g) (its buffer), then P.V(g) once
      // the softmax has stored P(g): the tensor pipe always holds the next logits
      if (s_ok) {
        issue_s(cs);
        advance(cs, s_ok, false);
      }
      const int vst = int(cp.g % kVST), ob = cp.oi & 1, pb = int(cp.g & 1);
      if (cp.t == 0 && cp.oi >= 2) mbar_wait(&bar_oempty[ob], ((cp.oi >> 1) + 1) & 1);
      mbar_wait(&bar_pfull[pb], (cp.g >> 1) & 1);
      if (lane == 0) KTR(cp.g, 6);
      mbar_wait(&bar_vfull[vst], (cp.g / kVST) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sV = smem_u32(smem + KtSmem::kV + vst * KtSmem::kPair);
        const bool single = (cp.t == cp.np - 1) && (cp.n & 1);
        const int nk = single ? 4 : 8;
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t ad = sdesc_sw128(sV + (kk >> 2) * 16384 + (kk & 3) * 2048, 8192, 1024);
          const uint64_t bd = sdesc_sw128(sP + pb * 16384 + kk * 2048, 8192, 1024);
          umma_f16_ss(tmem + 128 + ob * 64, ad, bd, idesc_o, (cp.t > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&bar_vempty[vst]);
        umma_commit(&bar_pempty[pb]);
        if (cp.t == cp.np - 1) umma_commit(&bar_ofull[ob]);
        KTR(cp.g, 7);
      }
      __syncwarp();
      advance(cp, p_ok, true);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    const int q4 = warp & 3;              // TMEM lane quarter
    const int cg = (warp - 4) >> 2;       // column group
    const int kl = q4 * 32 + lane;        // key lane in the pair (0..127)
    const int half = kl >> 6, kk = kl & 63;
    const uint32_t lane_addr = uint32_t(q4 * 32) << 16;
    const float sl2 = a.scale_log2;
    uint8_t* Pbuf = smem + KtSmem::kP;
    const uint32_t prow = smem_u32(Pbuf + kl * 128);  // this thread's key row of P^T (buffer 0)
    long long g = 0;
    int oi = 0;
    for (int it = 0;; ++it) {
      const int slot = it % kIR;
      mbar_wait(&bar_ifull[slot], (it / kIR) & 1);
      const KtItem& I = items[slot];
      const int n = I.n;
      if (n < 0) break;
      const int b = I.b, h = I.h, i = I.i, diag = I.diag;
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_iempty[slot]);
      const long long orow0 = (long long)(b * a.H + h) * a.L + (long long)i * kBS;
      const int np = (n + 1) / 2;
      const int ob = oi & 1;
      // per query column c of this thread: offset m (kept negated, log2 units) and
      // the partial row sum over this thread's keys, as float2 pairs
      float2 nm[CPT / 2], lp[CPT / 2];
#pragma unroll
      for (int c = 0; c < CPT / 2; ++c) {
        nm[c] = make_float2(0.f, 0.f);
        lp[c] = make_float2(0.f, 0.f);
      }
      const float2 sl2v = make_float2(sl2, sl2);
      for (int t = 0; t < np; ++t, ++g) {
        const int sb = int(g & 1);
        mbar_wait(&bar_sfull[sb], (g >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 128) KTR(g, 1);
        float2 x[CPT / 2];
        {
          uint32_t v[CPT];
          if constexpr (CPT == 32) {
            tmem_ld32(tmem + lane_addr + sb * 64 + cg * CPT, v);
          } else {
            tmem_ld16(tmem + lane_addr + sb * 64 + cg * CPT, *reinterpret_cast<uint32_t(*)[16]>(v));
          }
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < CPT / 2; ++c)
            x[c] = __ffma2_rn(make_float2(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1])), sl2v, nm[c]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_sfree[sb]);
        if (threadIdx.x == 128) KTR(g, 2);
        if (t == np - 1 && ((n & 1) || diag)) {
          // last pair: an odd count has only block a; the diagonal block (the last
          // selected one) is causal at token level: key kk <= query column
          const bool lane_valid = !((n & 1) && half == 1);
          const bool diag_lane = diag && (half == ((n & 1) ? 0 : 1));
#pragma unroll
          for (int c = 0; c < CPT / 2; ++c) {
            const int col = cg * CPT + 2 * c;
            if (!lane_valid || (diag_lane && kk > col)) x[c].x = -INFINITY;
            if (!lane_valid || (diag_lane && kk > col + 1)) x[c].y = -INFINITY;
          }
        }
        float tmax = -INFINITY;
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) tmax = fmaxf(tmax, fmaxf(x[c].x, x[c].y));
        const bool resc_any = named_bar_or(1, kSmThreads, t == 0 || tmax > kT);
        if (threadIdx.x == 128) KTR(g, 3);
        if (resc_any) {
          // exact column maxima over the 128 key lanes, then move the offsets (first
          // step of the item: set them); rescale row sums and O^T by 2^-delta
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            float v = (c & 1) ? x[c >> 1].y : x[c >> 1].x;
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
            v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
            if ((c & 31) == lane) red[q4][cg * CPT + c] = v;
          }
          named_bar_sync(2, kSmThreads);
          float f[CPT];
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int col = cg * CPT + c;
            const float cm = fmaxf(fmaxf(red[0][col], red[1][col]), fmaxf(red[2][col], red[3][col]));
            const float delta = t == 0 ? cm : fmaxf(cm, 0.f);
            f[c] = t == 0 ? 0.f : ex2_approx(-delta);
            if (c & 1) {
              nm[c >> 1].y -= delta;
              x[c >> 1].y -= delta;
              lp[c >> 1].y *= f[c];
            } else {
              nm[c >> 1].x -= delta;
              x[c >> 1].x -= delta;
              lp[c >> 1].x *= f[c];
            }
          }
          named_bar_sync(2, kSmThreads);  // red[] is reused by the next reduction
          if (t > 0) {
            // O^T columns of this thread's queries: wait for P.V(g-1), scale, store back
            mbar_wait(&bar_pempty[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tc_fence_after();
            uint32_t o[CPT];
            const uint32_t oaddr = tmem + lane_addr + 128 + ob * 64 + cg * CPT;
            if constexpr (CPT == 32) {
              tmem_ld32(oaddr, o);
            } else {
              tmem_ld16(oaddr, *reinterpret_cast<uint32_t(*)[16]>(o));
            }
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < CPT; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f[c]);
            if constexpr (CPT == 32) {
              US_TMEM_ST_X32(oaddr, o);
            } else {
              tmem_st16(oaddr, *reinterpret_cast<const uint32_t(*)[16]>(o));
            }
            tmem_st_wait();
            tc_fence_before();
          }
        }
        // exponentials -> packed P^T row (this thread's key), row-sum partials
        uint32_t packed[CPT / 2];
#pragma unroll
        for (int c = 0; c < CPT / 2; ++c) {
          const float2 p = make_float2(ex2_approx(x[c].x), ex2_approx(x[c].y));
          lp[c] = __fadd2_rn(lp[c], p);
          packed[c] = pack_bf16(p.x, p.y);
        }
        if (threadIdx.x == 128) KTR(g, 4);
        if (g >= 2) mbar_wait(&bar_pempty[g & 1], ((g >> 1) + 1) & 1);  // P.V(g-2) has read this P^T buffer
#pragma unroll
        for (int u = 0; u < CPT / 8; ++u) {
          const uint32_t chunk = uint32_t(cg * (CPT / 8) + u);
          st_shared_v4(prow + uint32_t(g & 1) * 16384u + ((chunk ^ uint32_t(kl & 7)) << 4), packed[4 * u], packed[4 * u + 1],
                       packed[4 * u + 2], packed[4 * u + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_pfull[g & 1]);
        if (threadIdx.x == 128) KTR(g, 5);
        if (threadIdx.x == 32 * (4 + NSM - 1)) KTR(g, 11);
      }
      // ---- epilogue: row sums, O^T / l -> bf16 O rows, lse
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        float v = (c & 1) ? lp[c >> 1].y : lp[c >> 1].x;
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if ((c & 31) == lane) red[q4][cg * CPT + c] = v;
      }
      named_bar_sync(2, kSmThreads);
      if (warp - 4 < 2) {  // 64 threads: one per query column
        const int col = (warp - 4) * 32 + lane;
        const float l = red[0][col] + red[1][col] + red[2][col] + red[3][col];
        colv[col] = 1.f / l;
      }
      // m of column col lives in the threads of column group col / CPT
      if (q4 == 0 && a.lse) {
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          if ((c & 31) == lane) {
            const int col = cg * CPT + c;
            const float l = red[0][col] + red[1][col] + red[2][col] + red[3][col];
            const float mc = (c & 1) ? -nm[c >> 1].y : -nm[c >> 1].x;
            a.lse[orow0 + col] = (mc + __log2f(l)) * 0.69314718055994531f;
          }
      }
      mbar_wait(&bar_ofull[ob], (oi >> 1) & 1);
      tc_fence_after();
      named_bar_sync(2, kSmThreads);  // colv ready; every warp is past its last P^T store
      {
        uint32_t o[CPT];
        const uint32_t oaddr = tmem + lane_addr + 128 + ob * 64 + cg * CPT;
        if constexpr (CPT == 32) {
          tmem_ld32(oaddr, o);
        } else {
          tmem_ld16(oaddr, *reinterpret_cast<uint32_t(*)[16]>(o));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_oempty[ob]);
        // stage O [64 queries][128 d] bf16 in the (now idle) P^T buffer, row stride 256 B
        __nv_bfloat16* st = reinterpret_cast<__nv_bfloat16*>(Pbuf);
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int col = cg * CPT + c;
          st[col * 128 + kl] = __float2bfloat16_rn(__uint_as_float(o[c]) * colv[col]);
        }
      }
      named_bar_sync(2, kSmThreads);
      {
        const uint4* s4 = reinterpret_cast<const uint4*>(Pbuf);
        uint4* d4 = reinterpret_cast<uint4*>(a.O + orow0 * 128);
        for (int e = threadIdx.x - 128; e < kBS * 128 / 8; e += kSmThreads) d4[e] = s4[e];
      }
      named_bar_sync(2, kSmThreads);  // staging read before the next item's P^T stores
      ++oi;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

us_status launch_attention_kt(const AttnArgs& a, const CUtensorMap& tmQ3, const CUtensorMap& tmK2,
                              const CUtensorMap& tmV3, cudaStream_t st) {
  if (a.D != 128) {
    set_error("attention (key-major kernel): d_k must be 128");
    return US_ERR_UNSUPPORTED;
  }
  if (a.N > kMaxN) {
    set_error("attention: N (=L/S) above 4096 is not supported on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  const int smem = KtSmem::kBytes + 1024;
  int dev = 0;
  US_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  int sms = 148;
  US_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
  const long long n_items = (long long)a.B * a.H * a.N;
  const int grid = int(n_items < sms ? n_items : sms);
  // softmax column groups (calibration knob US_ATTN_KT_NCG): 2 -> 8 softmax warps with
  // 32 query columns each, 4 -> 16 warps with 16 columns each
  static const int ncg = [] {
    const char* e = std::getenv("US_ATTN_KT_NCG");
    return (e && std::atoi(e) == 2) ? 2 : 4;
  }();
  if (ncg == 2) {
    static std::atomic<uint64_t> attr_done{0};
    if (us_status s = ensure_smem_attr(attn_kt_kernel<2>, smem, attr_done, "attn_kt_kernel smem attribute"); s != US_OK)
      return s;
    attn_kt_kernel<2><<<grid, 32 * (4 + 4 * 2), smem, st>>>(tmQ3, tmK2, tmV3, a);
  } else {
    static std::atomic<uint64_t> attr_done{0};
    if (us_status s = ensure_smem_attr(attn_kt_kernel<4>, smem, attr_done, "attn_kt_kernel smem attribute"); s != US_OK)
      return s;
    attn_kt_kernel<4><<<grid, 32 * (4 + 4 * 4), smem, st>>>(tmQ3, tmK2, tmV3, a);
  }
  US_LAUNCH_CHECK("attn_kt_kernel");
  return US_OK;
}

}  // namespace us

#if US_KT_TRACE
extern "C" int us_debug_kt_trace(int cta, long long* host_out) {
  if (host_out) return int(cudaMemcpyFromSymbol(host_out, ::g_kt_trace, sizeof(long long) * 4096 * 16));
  return int(cudaMemcpyToSymbol(::g_kt_trace_cta, &cta, sizeof(int)));
}
#endif
