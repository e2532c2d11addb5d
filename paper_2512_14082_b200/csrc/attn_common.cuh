// attn_common.cuh — pieces shared by the block-sparse attention kernels
// (attention.cu, attention_tp.cu): the CTA work decode (four query groups that
// read one KV head), the ascending union list of the groups' selected key blocks
// with each tile's own-step list, and the FMA-pipe exp2.
//
// Reference semantics: block_sparse_attention (attention.cpp:89-137) visits the
// selected key blocks j <= i of each (head, query block) in ascending order; the
// union list preserves that order for every group, and a group that did not
// select a union block contributes P = 0 rows there.
#pragma once
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace attn {

constexpr int kBS = 64;      // block size (keys per tile, rows per group)
constexpr int kMaxN = 4096;  // blocks per row
constexpr int kMaxW = kMaxN / 32;

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

// Work order: KV head outermost, query blocks heaviest-first inside it, so the
// ~148 resident CTAs all stream K/V of ONE KV head (L * d * 4 bytes = 64 MB at
// 128K, d=128) and their random selected-block reads hit the 126 MB L2.
struct Groups {
  int b, h[4], i[4];
  bool en[4];
};

// CTA = 4 groups (head, query block) that read the same KV head:
//   group_mode 0 (H/H_kv % 4 == 0): 4 consecutive heads of a KV group at one query block
//   group_mode 1 (H/H_kv == 2)    : both heads of the group at query blocks (i, i-1)
//   group_mode 2 (otherwise)      : one head at 4 consecutive query blocks
__device__ __forceinline__ Groups decode_item(const AttnArgs& a, int item) {
  Groups g;
  const int G = a.H / a.H_kv;
  if (a.group_mode == 0) {
    const int quads = a.H / 4;
    const int i = a.N - 1 - item % a.N;
    const int bq = item / a.N;
    g.b = bq / quads;
    const int h0 = (bq % quads) * 4;
    for (int k = 0; k < 4; ++k) {
      g.h[k] = h0 + k;
      g.i[k] = i;
      g.en[k] = true;
    }
  } else if (a.group_mode == 1) {
    const int npairs = (a.N + 1) / 2;
    const int ip = npairs - 1 - item % npairs;
    const int bk = item / npairs;
    g.b = bk / a.H_kv;
    const int h0 = (bk % a.H_kv) * G;
    const int ib = 2 * ip + 1, ia = 2 * ip;
    for (int k = 0; k < 4; ++k) {
      g.h[k] = h0 + (k & 1);
      g.i[k] = k < 2 ? ib : ia;
    }
    for (int k = 0; k < 4; ++k) g.en[k] = g.i[k] < a.N;
  } else {
    const int nq = (a.N + 3) / 4;
    const int iq = nq - 1 - item % nq;
    const int bh = item / nq;
    g.b = bh / a.H;
    for (int k = 0; k < 4; ++k) {
      g.h[k] = bh % a.H;
      g.i[k] = 4 * iq + 3 - k;
      g.en[k] = g.i[k] < a.N;
    }
  }
  return g;
}

inline long long work_items(const AttnArgs& a) {
  if (a.group_mode == 0) return (long long)a.B * (a.H / 4) * a.N;
  if (a.group_mode == 1) return (long long)a.B * a.H_kv * ((a.N + 1) / 2);
  return (long long)a.B * a.H * ((a.N + 3) / 4);
}

// The automatic kernel choice for a mask (a.sel_pairs set): the M = 64 chains of
// attention64.cu when under 55 % of the causal (i, j <= i) block pairs are selected, the
// two-tile kernel otherwise. Measured at C3 shapes, L = 64K (profiles/r02d/README.md):
// attention64 takes 0.80x the time of attn_kernel at 10.6 % selected, 0.86x at 32 %, 0.95x
// at 43 % and 50 %, 1.02x at 62 %, 1.07x at 81 %.
// Decided per (batch item, KV head) — a unit every split of a call preserves (batch items,
// the KV-head chunks of Engine.run_host), so a layer's output does not depend on how it
// was partitioned.
__device__ __forceinline__ bool m64_wins(const AttnArgs& a, int b, int kvh) {
  const unsigned long long pairs = (unsigned long long)(a.H / a.H_kv) * a.N * (a.N + 1) / 2;
  return a.sel_pairs[b * a.H_kv + kvh] * 20ull < pairs * 11ull;
}

__device__ __forceinline__ int last_block(const AttnArgs& a, const Groups& gr) {
  int jmax = -1;
  for (int k = 0; k < 4; ++k)
    if (gr.en[k]) jmax = max(jmax, a.noncausal ? a.N - 1 : gr.i[k]);
  return jmax;
}

// Shared-memory lists the builder warp writes.
struct ListsCore {
  uint32_t mrow[4][kMaxW];
  // union of the four groups' selected blocks, ascending: j | sel_slot << (12 + slot)
  uint16_t steps[kMaxN];
  int n_own[2];
  int n_steps;
  uint32_t perm;  // group of tile slot s = (perm >> 2s) & 3
};
struct Lists : ListsCore {
  // per tile: the union positions it computes (its own steps), ascending
  uint16_t own_pos[2][kMaxN];
};

// Next union position >= t that tile x computes (T past the last).
__device__ __forceinline__ int next_own(const ListsCore& ls, int x, int t, int T) {
  while (t < T && ((ls.steps[t] >> (12 + 2 * x)) & 3u) == 0u) ++t;
  return t;
}

// One warp: mask rows restricted to the causal prefix, the asynchronous data-error
// report, the tile pairing, the union list and the two own-step lists.
// `pairing` allows the union-size-minimising pairing of the four groups into tiles.
// own_pos (nullable): the per-tile own-step lists.
__device__ __forceinline__ void build_lists(const AttnArgs& a, const Groups& gr, int jmax, bool pairing,
                                            ListsCore& ls, uint16_t (*own_pos)[kMaxN]) {
  const int lane = threadIdx.x & 31;
  const int nw = jmax >= 0 ? (jmax >> 5) + 1 : 0;
  for (int g = 0; g < 4; ++g) {
    const int ig = gr.i[g];
    const uint32_t* src =
        a.mask ? a.mask + ((long long)(gr.b * a.planes + gr.h[g] / a.heads_per_plane) * a.N + ig) * a.W : nullptr;
    // (non-causal dense attention, dense_attention(in, false): every key block j < N)
    const int jlast = a.noncausal ? a.N - 1 : ig;
    for (int w = lane; w < nw; w += 32) {
      uint32_t word = 0;
      if (gr.en[g] && (w << 5) <= jlast) {
        word = src ? src[w] : ~0u;
        const int hi = jlast - (w << 5);  // bits 0..hi are attended
        if (hi < 31) word &= (2u << hi) - 1u;
      }
      ls.mrow[g][w] = word;
    }
  }
  __syncwarp();
  if (a.err && a.mask) {
    // asynchronous data-error report (the reference throws, attention.cpp:106-108,
    // 127-129): a non-causal bit anywhere in a group's row, or an empty causal prefix
    for (int g = 0; g < 4; ++g) {
      if (!gr.en[g]) continue;
      const int ig = gr.i[g];
      const long long row = (long long)(gr.b * a.planes + gr.h[g] / a.heads_per_plane) * a.N + ig;
      const uint32_t* src = a.mask + row * a.W;
      uint32_t bad = 0;
      int cnt = 0;
      for (int w = lane; w < a.W; w += 32) {
        const uint32_t word = src[w];
        const int lo = w << 5;
        const uint32_t keep = lo > ig ? 0u : (ig - lo >= 31 ? ~0u : (2u << (ig - lo)) - 1u);
        bad |= word & ~keep;
        cnt += __popc(word & keep);
      }
      bad = __reduce_or_sync(0xffffffffu, bad);
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0 && (bad || cnt == 0)) {
        atomicOr(a.err, bad ? 4u : 8u);
        atomicMin(a.first_bad, int32_t(row));
      }
    }
  }
  // Pair the four groups into the two tiles so that the LONGER tile's step count
  // (its pair's union) is smallest: the CTA lasts as long as its longer tile.
  // Ties keep the natural order.
  int c01 = 0, c23 = 0, c02 = 0, c13 = 0, c03 = 0, c12 = 0;
  for (int w = lane; w < nw; w += 32) {
    const uint32_t m0 = ls.mrow[0][w], m1 = ls.mrow[1][w], m2 = ls.mrow[2][w], m3 = ls.mrow[3][w];
    c01 += __popc(m0 | m1);
    c23 += __popc(m2 | m3);
    c02 += __popc(m0 | m2);
    c13 += __popc(m1 | m3);
    c03 += __popc(m0 | m3);
    c12 += __popc(m1 | m2);
  }
  c01 = __reduce_add_sync(0xffffffffu, c01);
  c23 = __reduce_add_sync(0xffffffffu, c23);
  c02 = __reduce_add_sync(0xffffffffu, c02);
  c13 = __reduce_add_sync(0xffffffffu, c13);
  c03 = __reduce_add_sync(0xffffffffu, c03);
  c12 = __reduce_add_sync(0xffffffffu, c12);
  int pr = 0, best = max(c01, c23) * 4096 + c01 + c23;
  const int k1 = max(c02, c13) * 4096 + c02 + c13, k2 = max(c03, c12) * 4096 + c03 + c12;
  if (pairing && k1 < best) {
    pr = 1;
    best = k1;
  }
  if (pairing && k2 < best) {
    pr = 2;
    best = k2;
  }
  // slot s (tile s / 2, rows (s & 1) * 64 ..) holds group perm[s]
  const uint32_t perm = pr == 0 ? 0xE4u : pr == 1 ? 0xD8u : 0x9Cu;  // 2-bit fields: 0123 / 0213 / 0312
  int base = 0;
  for (int w0 = 0; w0 < nw; w0 += 32) {
    const int w = w0 + lane;
    uint32_t m[4];
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) m[sl] = w < nw ? ls.mrow[(perm >> (2 * sl)) & 3u][w] : 0u;
    uint32_t u = m[0] | m[1] | m[2] | m[3];
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
      uint32_t e = uint32_t((w << 5) + bit);
#pragma unroll
      for (int g = 0; g < 4; ++g) e |= ((m[g] >> bit) & 1u) << (12 + g);
      ls.steps[pos++] = uint16_t(e);
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  // own-step counts (and lists) of the two tiles
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    int n = 0;
    for (int t0 = 0; t0 < base; t0 += 32) {
      const int t = t0 + lane;
      const bool mine = t < base && ((ls.steps[t] >> (12 + 2 * x)) & 3u) != 0u;
      const uint32_t b = __ballot_sync(0xffffffffu, mine);
      if (mine && own_pos) own_pos[x][n + __popc(b & ((1u << lane) - 1u))] = uint16_t(t);
      n += __popc(b);
    }
    if (lane == 0) ls.n_own[x] = n;
  }
  if (lane == 0) {
    ls.n_steps = base;
    ls.perm = perm;
  }
}

}  // namespace attn
}  // namespace us
