// kernels.cuh — launch interfaces of the hot-path kernels (device code lives in
// compress.cu, proxy.cu, select.cu, attention.cu). All launches are
// asynchronous on the given stream.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/us_api.h"

namespace us {

// ---------------------------------------------------------------- compress (a1)
// One output plane = mean over `members` source heads of the window means of
// `c` consecutive rows (compression.hpp:26-28 then :61-76), fp64 accumulation,
// one f32 rounding per stage. Source head of member g of plane p is
// (p * members + g) / div.
struct CompressArgs {
  const uint16_t* src;  // bf16 [B][H_src][L][d] (f32 when src_f32; reinterpreted)
  int B, H_src, L, d;
  int c;           // window (c_q or c_k)
  int planes;      // output planes per batch item
  int members;     // heads pooled per plane (c_h, or 1 when deduplicated)
  int div;         // member head -> source head divisor (G for expanded K, 1 for Q)
  float* out;      // f32 [B][planes][L/c][d]
  uint32_t* absmax;  // [B * planes] max |out| as f32 bits (may be null)
  int strategy;    // US_POOL_MEAN / MAX / STOCHASTIC (compression.hpp:24-53)
  int role;        // stochastic seed tag: 0 = Q, 1 = K (compression.cpp:17-20)
  uint64_t seed;   // CompressionConfig::seed
  int head0;       // global index of the call's first head (stochastic seeds use head0 + h)
  // fused split (nullable): fp16 hi/lo of out * 2^row_exp[row] per output row [B*planes][L/c][d]
  __half* hi;
  __half* lo;
  int* row_exp;    // [B*planes][L/c]
  int src_f32;     // 1: src holds f32 values (the reference's fp32 HeadStack storage)
};
us_status launch_compress(const CompressArgs& a, cudaStream_t st);

// f32 planes -> fp16 (hi, lo) pair scaled by 2^e (e per plane, from absmax) so
// that hi + lo carries ~22 significant bits for the fp16x3 tensor-core proxy.
struct SplitArgs {
  const float* in;  // [planes_total][rows][d]
  int planes_total, rows, d;
  const uint32_t* absmax;  // [planes_total]
  int* exp_out;            // [planes_total] scale exponents e
  __half* hi;
  __half* lo;
};
us_status launch_split(const SplitArgs& a, cudaStream_t st);
// f32 -> bf16 (round to nearest even) of n elements (n % 4 == 0): the bf16 copies
// attention computes on when the caller's Q/K/V are f32 (us_params.dtype).
us_status launch_f32_to_bf16(const float* in, void* out, long long n, cudaStream_t st);

// ---------------------------------------------------------------- proxy (a2-a3)
struct ProxyArgs {
  int B, Hc, Lq, Lk, N, D;
  int rq, rk;          // composite rows per query block, keys per key block
  int c_q, c_k;
  int causal_mode;
  int kv_planes;       // K planes per batch item
  int kv_mul, kv_div;  // K plane of compressed head hc = hc * kv_mul / kv_div
  const int* exp_q;    // [B*Hc][Lq] per composite row (q_row_exp = 1) or [B*Hc] per plane
  const int* exp_k;    // [B*kv_planes]
  const __half* qh;    // [B*Hc][Lq][D] fp16 hi of Qc * 2^e
  const __half* ql;    // [B*Hc][Lq][D] fp16 lo
  int T;               // key tiles of 128 composite keys = ceil(Lk / 128)
  int sw;              // slot width in composite keys = min(rk, 8)
  float* part;         // [B*Hc][T][Lq][128/sw] slot sums of 2^(x - tile max)
  float* tmax;         // [B*Hc][T][Lq] tile max (log2 units)
  float* lse2;         // [B*Hc][Lq] row log-sum-exp in log2 units
  float* scores;       // [B*Hc][N][N] block scores (j <= i)
  float scale_log2;    // log2(e) / sqrt(d_k)
  // competitor proxies (x3 = 0): raw bf16 rows of one phase class, single MMA
  int x3;              // 1: UniSparse fp16x3 on compressed rows; 0: bf16 raw rows
  const uint16_t* qraw;  // bf16 Q [B][Hc][L][D]
  int L;               // original sequence length (raw Q row stride per head)
  int q_row0, q_stride, q_phase;  // query composite row r -> raw row q_row0 + r*q_stride + q_phase
  int k_phase;         // key phase class (3-D K map: (d, stride, rows/stride))
  int live_bias;       // live keys of composite row r = r + live_bias
  int accumulate;      // finalize adds into scores instead of overwriting
  int q_row_exp;       // 1: exp_q holds one exponent per composite query row
  int finalize;        // 1: launch the finalize (block scores into `scores`); 0: the caller
                       //    fuses it into the selection (launch_select_fused)
};
int proxy_slot_width(int rk);
// One pass (logits, row LSE, slot partials) then the finalize (block scores).
us_status launch_proxy(const ProxyArgs& a, const CUtensorMap& tmKh, const CUtensorMap& tmKl,
                       cudaStream_t st);

// ---------------------------------------------------------------- last-block probe (competitor)
struct LastBlockArgs {
  int B, H, H_kv, L, N, D;
  const uint16_t* Q;   // bf16 [B][H][L][D]
  const uint16_t* K;   // bf16 [B][H_kv][L][D]
  float scale_log2;
  float* cmax;         // [B*H][L/256][64] chunk maxima (log2 units)
  float* csum;         // [B*H][L/256][64] chunk sums
  float* lse2;         // [B*H][64]
  float* colmass;      // [B*H][N]
  float* scores;       // [B*H][N][N] (j <= i)
};
us_status launch_last_block_probe(const LastBlockArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- selection (a4-a5)
struct SelectArgs {
  const float* scores;  // [rows][N] (row = (b*planes + p)*N + i), j <= i read
  float* scores_out;    // fused path: raw block scores written here when non-null
  int rows, N, W;
  int select_mode;
  double P;
  int top_k;
  uint32_t* mask_bits;  // [rows][W]
  int32_t* counts;      // [rows] (nullable)
  double* coverage;     // [rows] (nullable)
  int16_t* indices;     // [rows][N] (nullable)
  uint32_t* err;        // device error word (bit 0: negative/NaN score)
  int32_t* fb_count;    // fallback row counter
  int32_t* fb_rows;     // fallback row list [rows]
};
us_status launch_select(const SelectArgs& a, cudaStream_t st);
// Fused finalize + selection (UniSparse path): one CTA per (plane, query block)
// row builds the row's block scores in shared memory from the proxy's slot
// partials (proxy_score.cuh), selects by radix descent + fp64 certification, and
// emits bits / counts / coverage / indices; sa.scores_out (nullable) receives the raw
// scores when the caller asked for them. Uncertified rows go to the exact
// sorted-walk fallback, which recomputes the row from the partials.
us_status launch_select_fused(const ProxyArgs& pa, const SelectArgs& sa, cudaStream_t st);

// ---------------------------------------------------------------- attention (a6)
struct AttnArgs {
  int B, H, H_kv, L, N, W, D;
  int group_mode;       // CTA groups: 0 = 4 heads of a KV group, 1 = 2 heads x 2 blocks, 2 = 1 head x 4 blocks
  int heads_per_plane;  // mask plane of head h = h / heads_per_plane
  int planes;           // mask planes per batch item
  const uint32_t* mask; // [B][planes][N][W] (nullptr = dense causal)
  const __nv_bfloat16* Q; // [B][H][L][D] (rows go straight to TMEM)
  __nv_bfloat16* O;     // [B][H][L][D]
  float* lse;           // [B][H][L] (nullable)
  float scale_log2;
  int pairing;          // 1: pair the CTA's groups into tiles by union size (0: fixed 01|23)
  int one_tile;         // 1: one M=128 tile (two groups) per CTA, two CTAs per SM
  uint32_t* err;        // device error word (nullable): |= 4 non-causal bit, |= 8 empty row
  int32_t* first_bad;   // first offending mask row (atomicMin; nullable with err)
  int noncausal;        // 1: dense_attention(in, causal = false): all N key blocks, no diagonal mask
  int32_t* items;       // attention64.cu: work-item table [B*H_kv][ceil(G*N/4)][4] of (h << 16 | i), -1 = none
                        // (nullable: the fixed decode_item order)
  int32_t* row_counts;   // attention64.cu: selected blocks j <= i per mask row [B][planes][N] (with a.items)
  unsigned long long* sel_pairs;  // automatic choice (nullable = off): selected (i, j <= i) pairs of the mask
                                  // per (batch item, KV head) [B][H_kv], summed by attn64_counts_kernel; both
                                  // kernels are launched and each CTA exits unless attn::m64_wins picks its
                                  // kernel for its (b, KV head) (attn_common.cuh)
};
us_status launch_attention(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                           const CUtensorMap& tmV, cudaStream_t st);

// Decoupled-softmax variant (attention_tp.cu): same work decomposition and union lists
// as launch_attention; two logit buffers per tile in TMEM, P written back into them and
// P.V as a TS-mode MMA, Q in SMEM (SS-mode S), two softmax warps per lane quarter.
// tmQ: 2-D map (box 64 rows x 64); tmK / tmV: 3-D rows-chunked maps (box 64 rows).
us_status launch_attention_tp(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK,
                              const CUtensorMap& tmV, cudaStream_t st);

// One M = 64 UMMA chain per query group (attention64.cu): same work decomposition and
// union list as launch_attention, two groups per set of TMEM columns at lane offsets 0 / 16.
// tmK / tmV: 3-D rows-chunked maps (box 64 rows).
us_status launch_attention64(const AttnArgs& a, const CUtensorMap& tmQ, const CUtensorMap& tmK, const CUtensorMap& tmV,
                             cudaStream_t st);
// int32 entries of the attention64 work-item table (a.items) for these dims, and the bytes
// of its workspace region: [item table][sel_pairs: B * H_kv u64][row_counts: B * H * N int32]
long long attention64_item_entries(int B, int H, int H_kv, int N);
size_t attention64_ws_bytes(int B, int H, int H_kv, int N);

// Key-major variant (attention_kt.cu, d_k = 128): one query group per work item,
// M = 128 = a pair of its own selected key blocks (no union rows); persistent CTAs.
// tmQ3 / tmV3: 3-D rows-chunked maps (box 64 rows), tmK2: 2-D map (box 64 x 64).
us_status launch_attention_kt(const AttnArgs& a, const CUtensorMap& tmQ3, const CUtensorMap& tmK2,
                              const CUtensorMap& tmV3, cudaStream_t st);

// 128-key-step variant (attention2.cu): one M=128 tile per CTA, two union blocks
// per step; Q is read from global memory by the softmax warps (no Q tensor map).
us_status launch_attention2(const AttnArgs& a, const CUtensorMap& tmK, const CUtensorMap& tmV,
                            cudaStream_t st);

// ---------------------------------------------------------------- quality metrics (metrics.cu)
us_status launch_fill_upper(float* scores, long long planes, int N, cudaStream_t st);
us_status launch_planted_recall(int B, int H, int N, int W, int planes, int heads_per_plane, int m,
                                const uint32_t* mask, const int32_t* planted, double* rows_ws, uint8_t* defined,
                                double* out, long long* n_def, cudaStream_t st);
us_status launch_output_fidelity(long long rows, int d, const uint16_t* test, const uint16_t* ref, double* rows_ws,
                                 double* out3, cudaStream_t st);
us_status launch_block_recall(int B, int H, int N, int W, int planes, int heads_per_plane, int k,
                              const uint32_t* mask, const float* ref, double* rows_ws, double* out,
                              cudaStream_t st);
us_status launch_row_spearman(int B, int H, int N, int c_h, const float* proxy, const float* ref, double* rows_ws,
                              uint8_t* defined, double* out, long long* n_def, cudaStream_t st);

// S = 64 m block masks [planes][N][W] -> 64-granular masks [planes][N m][ceil(N m / 32)]
// (sub-blocks of the diagonal block wholly in the future dropped), for the attention kernels.
us_status launch_mask_expand(const uint32_t* in, long long planes, int N, int W, int m, uint32_t* out,
                             cudaStream_t st);

// mask validation: err |= 4 for a non-causal bit, 8 for an empty causal row;
// first offending row index (b*planes+p)*N+i recorded with atomicMin in *first_bad.
us_status launch_mask_check(const uint32_t* mask, int rows, int N, int W, uint32_t* err,
                            int32_t* first_bad, cudaStream_t st);

}  // namespace us
