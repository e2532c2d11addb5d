/*
 * us_api.h — C ABI of the B200-native UniSparse hot path (sm_100a).
 *
 * Drop-in boundary for the reference operator API (namespace unisparse,
 * /root/reference/proj/include/unisparse/):
 *
 *   reference (C++, by value, exceptions)              this ABI (C, device pointers, status)
 *   -------------------------------------------------  -----------------------------------------
 *   compress(in, cfg)            compression.hpp:89    us_compress
 *   select_blocks(UniSparse, in, cfg) pipeline.hpp:19  us_select
 *   build_block_mask(scores,P,c_h,H) selection.hpp:41  us_build_block_mask
 *   block_sparse_attention(in, mask) attention.hpp:27  us_sparse_attention
 *   unisparse_attn(in, cfg)      pipeline.hpp:16       us_unisparse_attention
 *   dense_attention(in, causal)  attention.hpp:16      us_dense_attention (+ US_FLAG_NONCAUSAL)
 *   validate_inputs(in, cfg)     types.hpp:106         us_validate
 *   selection_flops(...)         metrics.hpp:31        us_selection_flops
 *   CompressionConfig / AttentionInputs types.hpp:54-72  us_params
 *
 * Conventions
 *   * Tensors are device pointers, head-major (the reference HeadStack order,
 *     tensor_io.hpp:9-11) with a leading batch dim:
 *       Q, O      bf16 [B][H][L][d_k]   (Q / K / V f32 when params.dtype = US_DTYPE_F32)
 *       K, V      bf16 [B][H_kv][L][d_k]   (GQA: head h reads KV head h/(H/H_kv);
 *                                          H_kv == H is the reference layout)
 *       lse       f32  [B][H][L]           natural log, reference AttentionOutput::lse
 *   * Selection planes: one plane per compressed head (H/c_h planes); head h
 *     uses plane h / c_h (the broadcast of selection.cpp:80-84).
 *       mask_bits u32  [B][planes][N][W], W = ceil(N/32); bit (j%32) of word
 *                 j/32 in row i set <=> key block j is attended by query block i.
 *   * No allocation inside timed calls: the caller passes a workspace of at
 *     least us_workspace_bytes(params) bytes (device memory).
 *   * `stream` is a cudaStream_t (void* keeps CUDA headers out of this file).
 *     Calls are asynchronous unless US_FLAG_SYNC_CHECK is set in params.flags,
 *     in which case the call synchronizes the stream and reports data errors
 *     (negative/NaN proxy scores, malformed masks) the way the reference throws.
 *   * No C++ exceptions cross this boundary. Errors return a us_status and set
 *     a thread-local message (us_last_error) carrying the reference's text,
 *     e.g. "select_blocks: L=1000 not divisible by S=64".
 *   * Reentrant: no global mutable state besides per-thread error text and
 *     per-device one-time init (std::call_once).
 */
#ifndef US_API_H
#define US_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum us_status {
  US_OK = 0,
  US_ERR_INVALID_ARGUMENT = 1, /* shapes / config: reference std::invalid_argument */
  US_ERR_UNSUPPORTED = 2,      /* valid for the reference, not on this GPU path (e.g. d_k=96) */
  US_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  US_ERR_INVALID_MASK = 4,     /* non-causal bit or empty row (attention.cpp:106-108,127-129) */
  US_ERR_NONFINITE = 5,        /* negative/NaN proxy scores (selection.cpp:14-15) */
  US_ERR_WORKSPACE = 6,        /* workspace missing or too small */
  US_ERR_IO = 7                /* file I/O: reference std::runtime_error (tensor_io.cpp:15-17) */
} us_status;

/* PoolStrategy (types.hpp:34) — the GPU path implements Mean. */
enum { US_POOL_MEAN = 0, US_POOL_MAX = 1, US_POOL_STOCHASTIC = 2 };
/* CausalMode (types.hpp:36-42) */
enum { US_POST_SOFTMAX_BLOCK_CAUSAL = 0, US_PRE_SOFTMAX_COMPRESSED_CAUSAL = 1 };
/* selection rule: reference Top-P (selection.cpp:11-48), or top-k = first k of the same order */
enum { US_SELECT_TOP_P = 0, US_SELECT_TOP_K = 1 };
/* ProxyTag (types.hpp:45) for us_selection_flops */
enum { US_PROXY_UNISPARSE = 0, US_PROXY_ANTIDIAGONAL = 1, US_PROXY_LAST_BLOCK = 2 };
/* params.dtype */
enum { US_DTYPE_BF16 = 0, US_DTYPE_F32 = 1 };
/* params.flags */
enum { US_FLAG_SYNC_CHECK = 1, US_FLAG_NONCAUSAL = 2 /* us_dense_attention: causal = false */ };

/* CompressionConfig (types.hpp:54-62) + AttentionInputs dims (types.hpp:66-72)
 * + the GQA / batch / top-k extensions the north star adds. */
typedef struct us_params {
  int32_t B;           /* batch */
  int32_t H;           /* query heads */
  int32_t H_kv;        /* key/value heads (H % H_kv == 0) */
  int32_t L;           /* sequence length (L % S == 0) */
  int32_t d_k;         /* head dim (GPU path: 64 or 128) */
  int32_t S;           /* block size (GPU path: 64) */
  int32_t c_q, c_k, c_h;
  int32_t strategy;    /* US_POOL_* */
  int32_t causal_mode; /* US_POST_SOFTMAX_BLOCK_CAUSAL (reference default) or pre */
  int32_t select_mode; /* US_SELECT_TOP_P / US_SELECT_TOP_K */
  double P;            /* Top-P mass threshold in (0, 1], kept in double (types.hpp:59) */
  int32_t top_k;       /* k for US_SELECT_TOP_K */
  int32_t flags;       /* US_FLAG_* */
  uint64_t seed;       /* stochastic pooling seed (unused by Mean) */
  int32_t dtype;       /* US_DTYPE_BF16 (0, default) or US_DTYPE_F32: storage of Q, K, V.
                          F32 is the reference's own HeadStack<float> (types.hpp:15-26):
                          compress / select pool the f32 values (fp64 window sums,
                          compression.hpp:26-28); attention computes on bf16 copies made
                          in the workspace (O stays bf16). */
  int32_t head0;       /* global index of this call's first Q head (0 for a whole layer): a
                          call on a head range [head0, head0 + H) of a larger layer (head
                          sharding, chunked pipelines) seeds stochastic pooling with the
                          global head index, as the reference does (compression.cpp:17-20) */
} us_params;

/* Selection outputs (device pointers; every field except mask_bits may be NULL).
 * The reference SparsityReport (metrics.hpp:77-83) is derived from counts. */
typedef struct us_selection {
  uint32_t* mask_bits; /* [B][planes][N][W] */
  int32_t* counts;     /* [B][planes][N] selected blocks per row */
  double* coverage;    /* [B][planes][N] covered score fraction (BlockMask::coverage) */
  float* scores;       /* [B][planes][N][N] proxy block scores, j <= i written */
  int16_t* indices;    /* [B][planes][N][N] ascending selected block ids, counts[] valid */
} us_selection;

const char* us_version(void);
const char* us_last_error(void);

/* validate_inputs (types.cpp:97-123) plus GPU-path constraints. Returns the
 * number of violations; msg receives them joined by "; ". */
int us_validate(const us_params* p, char* msg, size_t cap);

/* The host-side gate every call below runs first, exposed so wrappers can
 * raise before allocating: US_OK, US_ERR_INVALID_ARGUMENT (reference
 * validate_inputs violations, text "<who>: v1; v2", types.cpp:97-123) or
 * US_ERR_UNSUPPORTED (GPU-path limits); message via us_last_error().
 * need_compression = 0 skips the compression-only limits (attention calls). */
us_status us_check_params(const us_params* p, const char* who, int32_t need_compression);

/* Device workspace needed by any call below for these params. */
size_t us_workspace_bytes(const us_params* p);

/* The smaller workspace that suffices for us_sparse_attention / us_dense_attention
 * (error header, bf16 copies of f32 inputs, the 64-granular mask for S > 64, the sparse
 * kernel's work-item table, zero-padded d_k copies) — no proxy / selection buffers,
 * which at the attention calls' c = 1 would scale with the uncompressed length. With
 * at least this many bytes the attention calls report mask errors asynchronously
 * (us_check_device_errors) and the density-gated sparse kernel runs. */
size_t us_attention_workspace_bytes(const us_params* p);

/* compress (compression.cpp:5-25), Mean pooling: Qc f32 [B][H/c_h][L/c_q][d_k],
 * Kc f32 [B][H/c_h][L/c_k][d_k] (K expanded to H heads first, as the reference). */
us_status us_compress(const us_params* p, const void* Q, const void* K, float* Qc, float* Kc,
                      void* workspace, size_t workspace_bytes, void* stream);

/* select_blocks (pipeline.cpp:5-17): compress -> proxy -> Top-P/top-k selection. */
us_status us_select(const us_params* p, const void* Q, const void* K, const us_selection* out,
                    void* workspace, size_t workspace_bytes, void* stream);

/* select_blocks(proxy, in, cfg, stride) (pipeline.cpp:5-17) for any proxy tag:
 * US_PROXY_UNISPARSE = us_select; US_PROXY_ANTIDIAGONAL = the XAttention-style
 * strided anti-diagonal scorer (antidiagonal_block_scores, baselines.cpp:10-52),
 * US_PROXY_LAST_BLOCK = the FlexPrefill-style last-block probe
 * (last_block_probe_scores, baselines.cpp:54-87); both per original head
 * (planes = H, no head compression, pipeline.cpp:11). The workspace must hold
 * us_proxy_workspace_bytes(p, proxy, stride) bytes. */
us_status us_select_proxy(const us_params* p, int32_t proxy, int32_t stride, const void* Q, const void* K,
                          const us_selection* out, void* workspace, size_t workspace_bytes, void* stream);
size_t us_proxy_workspace_bytes(const us_params* p, int32_t proxy, int32_t stride);

/* build_block_mask (selection.cpp:60-88) on given f32 block scores
 * [B][planes][N][N] (only j <= i read). */
us_status us_build_block_mask(const us_params* p, const float* scores, const us_selection* out,
                              void* workspace, size_t workspace_bytes, void* stream);

/* block_sparse_attention (attention.cpp:89-137). heads_per_plane maps head h to
 * mask plane h / heads_per_plane (1 = one plane per head, as the reference). */
us_status us_sparse_attention(const us_params* p, const void* Q, const void* K, const void* V,
                              const uint32_t* mask_bits, int32_t heads_per_plane, void* O,
                              float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* unisparse_attn (pipeline.cpp:19-24). sel may be NULL; if given, its non-NULL
 * fields receive the selection (mask_bits is then also used by attention). */
us_status us_unisparse_attention(const us_params* p, const void* Q, const void* K, const void* V,
                                 void* O, float* lse, const us_selection* sel, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* dense_attention(in, causal) (attention.cpp:20-54): the same kernel with every
 * causal block selected (the P = 1 path; reference criterion 1), or with every
 * key block and no diagonal mask when params.flags has US_FLAG_NONCAUSAL. */
us_status us_dense_attention(const us_params* p, const void* Q, const void* K, const void* V,
                             void* O, float* lse, void* workspace, size_t workspace_bytes,
                             void* stream);

/* ---- quality metrics on GPU outputs: the reference's
 * metrics.cpp:100-224 as used by run_experiment (experiment.cpp:280-437).
 * Scalar results go to HOST pointers; these calls synchronize the stream. */

/* exact_block_mass (attention.cpp:56-86): for head h and query block i, the mass
 * of the token-level causal softmax of Q_h K_{h/G}^T / sqrt(d_k) on key block j
 * (bf16 products, fp32 accumulation), f32 [B][H][N][N]; j > i holds the
 * reference's kMaskedScore (-FLT_MAX, types.hpp:32). The
 * workspace must hold us_mass_workspace_bytes(p) bytes (it grows as H * L^2). */
us_status us_exact_block_mass(const us_params* p, const void* Q, const void* K, float* mass, void* workspace,
                              size_t workspace_bytes, void* stream);
size_t us_mass_workspace_bytes(const us_params* p);

/* Workspace of the three metric calls below for these params. */
size_t us_metrics_workspace_bytes(const us_params* p);

/* output_fidelity (metrics.cpp:118-153) of bf16 O_test against bf16 O_ref, both
 * [B][H][L][d_k]: out3 = {max_abs, mean_rel, cosine} (fp64, the reference's
 * per-row sequential sums). */
us_status us_output_fidelity(const us_params* p, const void* O_test, const void* O_ref, double* out3,
                             void* workspace, size_t workspace_bytes, void* stream);

/* block_recall (metrics.cpp:155-176): mask planes [B][H/heads_per_plane][N][W]
 * against reference block scores ref f32 [B][H][N][N]; k in [1, N]. */
us_status us_block_recall(const us_params* p, const uint32_t* mask_bits, int32_t heads_per_plane, const float* ref,
                          int32_t k, double* out, void* workspace, size_t workspace_bytes, void* stream);

/* planted_recall (metrics.cpp:178-199): the mean over (b, h, i) rows with a
 * non-empty planted list of the fraction of planted blocks the mask selected;
 * planted int32 [B][H][N][m], -1 = unused slot (the generator's planted sets,
 * workloads.cpp:98-125). US_ERR_INVALID_ARGUMENT "planted_recall: no planted rows"
 * when every list is empty. */
us_status us_planted_recall(const us_params* p, const uint32_t* mask_bits, int32_t heads_per_plane,
                            const int32_t* planted, int32_t m, double* out, void* workspace, size_t workspace_bytes,
                            void* stream);

/* mean_row_spearman (metrics.cpp:201-224): proxy scores f32 [B][H/c_h][N][N]
 * (c_h = p->c_h) against ref f32 [B][H][N][N], rows i >= 1; flat rows count as
 * undefined. */
us_status us_mean_row_spearman(const us_params* p, const float* proxy, const float* ref, double* mean,
                               int64_t* defined, int64_t* undefined, void* workspace, size_t workspace_bytes,
                               void* stream);

/* Reads and clears the device-side data-error word of a workspace
 * (synchronizes the stream). */
us_status us_check_device_errors(const us_params* p, void* workspace, void* stream);

/* selection_flops (metrics.cpp:44-81): out6 = compression, compressed_qk,
 * softmax_aggregation, top_p, sparse_attention (0), dense_attention. */
us_status us_selection_flops(const us_params* p, int32_t proxy, int32_t stride, uint64_t* out6);

/* Block-sparse attention kernel used by every call in this process:
 * 0 = automatic (default, = 1); 1 = attention.cu (two M=128 query tiles per CTA, 64-key steps),
 * 2 = attention2.cu (one tile per CTA, 128-key steps), 3 = attention.cu with one
 * tile (two query groups) per CTA and two CTAs per SM, 4 = attention_kt.cu (key
 * blocks as the MMA M dimension, one query group per work item; d_k = 128), 5 = attention_tp.cu
 * (P in TMEM, two logit buffers per tile, Q in SMEM, split K / V rings). 2-5 exist only in the
 * calibration build. All compute the same function; the environment variable
 * US_ATTN_IMPL sets the initial choice. */
us_status us_set_attention_impl(int32_t impl);

/* Tile pairing inside an attention.cu CTA (calibration knob, process-wide):
 * 1 = pair the CTA's four query groups into its two M=128 tiles so that the
 * longer tile's step count is smallest (default), 0 = fixed pairing (01|23).
 * Outputs are bit-identical either way; the environment variable
 * US_ATTN_PAIRING sets the initial choice. */
us_status us_set_attention_pairing(int32_t on);

/* Number of kernel launches the last successful call on this thread issued. */
int32_t us_last_launch_count(void);

/* Per-stage CUDA-event timing (observability). While enabled, each
 * us_unisparse_attention call on this thread records events on its stream at
 * the stage boundaries [compress+split | proxy | select | attention] into the
 * next of `max_calls` slots. us_profile_read synchronizes on the recorded
 * events and writes [calls][4] stage times in ms; returns the number of calls. */
us_status us_profile_enable(int32_t max_calls);
int32_t us_profile_read(float* ms_out, int32_t max_calls);
void us_profile_disable(void);

/* ---- on-disk formats of the reference (host memory, no CUDA calls) ----------
 * unisparse.tn tensors (tensor_io.hpp:9-14; write_tensor / read_tensor,
 * tensor_io.cpp:31-81): 12-byte magic "unisparse.tn", u32 version 1, u32 H, L,
 * d_k, then H*L*d_k little-endian f32, head major. Errors carry the reference
 * text ("tensor file <path>: bad magic at offset 0", "payload shorter than
 * header H*L*d_k at offset ...", "trailing bytes beyond header H*L*d_k"). */
us_status us_write_tensor(const char* path, const float* data, int32_t H, int32_t L, int32_t d_k);
us_status us_read_tensor_header(const char* path, int32_t* H, int32_t* L, int32_t* d_k);
us_status us_read_tensor(const char* path, float* out, size_t capacity_floats);

/* RLE block-mask JSON (save_mask_json / load_mask_json, selection.cpp:90-144),
 * byte-identical to the reference's nlohmann dump(1, '\t'). mask_bits: host
 * [H/c_h][N][ceil(N/32)] planes, broadcast to the H heads. us_load_mask_json
 * fills H, N, P and, when out_bits is non-NULL, per-head bits [H][N][ceil(N/32)]. */
us_status us_save_mask_json(const char* path, const uint32_t* mask_bits, int32_t H, int32_t N, int32_t c_h,
                            double P);
us_status us_load_mask_json(const char* path, int32_t* H, int32_t* N, double* P, uint32_t* out_bits,
                            size_t capacity_words);

#ifdef __cplusplus
}
#endif

#endif /* US_API_H */
