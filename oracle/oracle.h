/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A CPU restatement ("ref64") of the UniSparse reference hot path
 * (/root/reference/proj, C++20 + Eigen), used as the parity checker for the
 * B200 kernels and as the bench's cpu_baseline leg. Nothing in the product
 * package (paper_2512_14082_b200/) may link, import or call this library.
 *
 * Why a restatement: the reference itself cannot be built in this container
 * (Eigen3 >= 3.3 and proj/vendor/ are absent; proj/CMakeLists.txt:12 fails).
 * Eigen's internal summation / exp order is therefore not reproduced
 * ("bitwise parity with the Eigen binary: unpinned"). What IS pinned: every
 * known-answer test the reference's own suite holds for this path
 * (tests/test_compression.cpp, test_proxy.cpp, test_selection.cpp,
 * test_attention.cpp, test_pipeline.cpp, test_metrics.cpp FLOP integers),
 * ported as pytest cases in tests/test_oracle_kat.py.
 *
 * Semantics followed (file:line in /root/reference/proj):
 *   RNG                 include/unisparse/rng.hpp:11-67
 *   workloads           src/workloads.cpp:18-128 (+ GQA extension, see .cpp)
 *   validation          src/types.cpp:97-123
 *   pool_sequence/heads include/unisparse/compression.hpp:13-76
 *   compress            src/compression.cpp:5-25
 *   compressed_attention src/proxy.cpp:10-46
 *   block_aggregate     src/proxy.cpp:48-72
 *   antidiagonal_block_scores, last_block_probe_scores  src/baselines.cpp:10-87
 *   top_p_row           src/selection.cpp:11-48
 *   build_block_mask    src/selection.cpp:60-88
 *   dense_attention     src/attention.cpp:20-54
 *   exact_block_mass    src/attention.cpp:56-87
 *   block_sparse_attention src/attention.cpp:89-137
 *   selection_flops etc src/metrics.cpp:44-151, 226-237
 *
 * Layouts: head-major, row-major within a head: X[h][t][c] (tensor_io.hpp:9-11).
 * GQA: K/V hold Hkv heads; Q head h reads K/V head h / (H / Hkv). With
 * Hkv == H this is exactly the reference. Masks are H planes of N*N bytes.
 * Return value: 0 on success, nonzero on error (message via or_last_error()).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_POOL_MEAN = 0, OR_POOL_MAX = 1, OR_POOL_STOCHASTIC = 2 };
enum { OR_POST_SOFTMAX = 0, OR_PRE_SOFTMAX = 1 };
enum { OR_SELECT_TOP_P = 0, OR_SELECT_TOP_K = 1 };
enum { OR_WL_GAUSSIAN = 0, OR_WL_PLANTED = 1, OR_WL_LOCALITY_SHIFT = 2 };
enum { OR_PROXY_UNISPARSE = 0, OR_PROXY_ANTIDIAGONAL = 1, OR_PROXY_LAST_BLOCK = 2 };

typedef struct or_cfg {
  int H, H_kv, L, d_k, S;
  int c_q, c_k, c_h;
  int strategy;
  int causal_mode;
  int select_mode;
  double P;
  int top_k;
  uint64_t seed;
} or_cfg;

const char* or_last_error(void);

/* --- RNG (rng.hpp) --- */
uint64_t or_mix64(uint64_t z);
uint64_t or_chain_seed(uint64_t seed, uint64_t tag);
/* n successive CounterRng(stream_seed) draws: kind 0 = next_u64, 1 = next_double,
 * 2 = next_double_open, 3 = next_gaussian (as double bit patterns for 1..3). */
void or_rng_draws(uint64_t stream_seed, int kind, int n, uint64_t* out);

/* --- workloads (workloads.cpp) --- planted: [H][N][m] block ids, -1 padded. */
int or_gen_workload(int kind, int L, int H, int H_kv, int d_k, int S, uint64_t seed,
                    double sigma, double gain, int m, float* Q, float* K, float* V,
                    int32_t* planted, int nthreads);

/* --- validation (types.cpp:97-123); writes the joined message, returns #errors --- */
int or_validate(const or_cfg* cfg, char* msg, int cap);

/* --- compression --- */
int or_pool_sequence(const float* x, int rows, int cols, int c, int strategy, uint64_t seed,
                     float* out);
/* Qc: [H/c_h][L/c_q][d], Kc: [H/c_h][L/c_k][d] (K expanded to H heads first). */
int or_compress(const or_cfg* cfg, const float* Q, const float* K, float* Qc, float* Kc);

/* --- proxy: block scores [H/c_h][N][N] (f64; j > i = kMaskedScore) --- */
int or_proxy_scores(const or_cfg* cfg, const float* Qc, const float* Kc, double* scores,
                    double* A_out, int nthreads);
/* Same scores but only for the listed query blocks of one compressed head:
 * out[r][N] for qblocks[r]. Cost O(rows * L/c_k * d): used for spot checks. */
int or_proxy_score_rows(const or_cfg* cfg, const float* Qc, const float* Kc, int hc,
                        const int32_t* qblocks, int nrows, double* out, int nthreads);

/* --- competitor proxies (baselines.cpp:10-87), H planes [H][N][N], j > i = kMaskedScore --- */
int or_antidiagonal_block_scores(int H, int H_kv, int L, int d_k, int S, int stride, const float* Q,
                                 const float* K, double* scores, int nthreads);
int or_last_block_probe_scores(int H, int H_kv, int L, int d_k, int S, const float* Q, const float* K,
                               double* scores, int nthreads);

/* --- selection --- */
int or_top_p_row(const double* scores, int n, double P, int32_t* indices, int* count,
                 double* covered);
int or_top_k_row(const double* scores, int n, int k, int32_t* indices, int* count,
                 double* covered);
/* mask: [H][N][N] bytes, coverage [H][N]. scores hold H/c_h planes. */
int or_build_block_mask(const double* scores, int H, int N, int c_h, int select_mode,
                        double P, int top_k, uint8_t* mask, double* coverage);

/* --- attention --- */
int or_dense_attention(int H, int H_kv, int L, int d_k, const float* Q, const float* K,
                       const float* V, int causal, float* O, double* lse, int nthreads);
int or_exact_block_mass(int H, int H_kv, int L, int d_k, int S, const float* Q,
                        const float* K, double* mass, int nthreads);
int or_block_sparse_attention(int H, int H_kv, int L, int d_k, int S, const float* Q,
                              const float* K, const float* V, const uint8_t* mask, float* O,
                              double* lse, int nthreads);
/* Sparse attention restricted to listed (head, query block) pairs; O rows for
 * pair r land at O[r][S][d], lse at lse[r][S]. */
int or_block_sparse_attention_rows(int H, int H_kv, int L, int d_k, int S, const float* Q,
                                   const float* K, const float* V, const uint8_t* mask,
                                   const int32_t* heads, const int32_t* qblocks, int nrows,
                                   float* O, double* lse, int nthreads);

/* --- metrics (metrics.cpp) --- out: compression, compressed_qk, softmax_aggregation,
 * top_p, sparse_attention(0), dense_attention. */
int or_selection_flops(uint64_t L, uint64_t H, uint64_t d_k, uint64_t S, int c_q, int c_k,
                       int c_h, int proxy, uint64_t stride, uint64_t* out6);
/* fidelity: out3 = max_abs, mean_rel, cosine */
int or_output_fidelity(const float* test, const float* ref, int H, int L, int d_k,
                       double* out3);

/* --- full pipeline (pipeline.cpp:19-24) for CPU timing --- */
/* metrics.cpp:100-224 — spearman_rho (average ranks), block_recall, mean_row_spearman */
int or_spearman_rho(const double* a, const double* b, int n, double* rho, int* defined);
int or_block_recall(const uint8_t* mask, const double* ref, int H, int N, int k, double* out);
int or_planted_recall(const uint8_t* mask, const int32_t* planted, int H, int N, int m, double* out);
int or_mean_row_spearman(const double* proxy, const double* ref, int H, int N, int c_h, double* mean,
                         int64_t* defined, int64_t* undefined);
int or_unisparse_attn(const or_cfg* cfg, const float* Q, const float* K, const float* V,
                      float* O, double* lse, uint8_t* mask, double* coverage, int nthreads);

#ifdef __cplusplus
}
#endif
