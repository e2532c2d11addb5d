/*
 * unisparse_b200.hpp — C++ mirror of the reference operator API over the C ABI.
 *
 * Header-only. Same names, argument meaning and error behaviour as the
 * reference (namespace unisparse, /root/reference/proj/include/unisparse/):
 *
 *   compress(in, cfg)                 compression.hpp:89   -> us_compress
 *   select_blocks(in, cfg)            pipeline.hpp:19-20   -> us_select
 *   build_block_mask(scores, cfg, H)  selection.hpp:41     -> us_build_block_mask
 *   block_sparse_attention(in, mask)  attention.hpp:27     -> us_sparse_attention
 *   unisparse_attn(in, cfg)           pipeline.hpp:16      -> us_unisparse_attention
 *   dense_attention(in)               attention.hpp:21     -> us_dense_attention
 *   selection_flops(...)              metrics.hpp:31       -> us_selection_flops
 *
 * Differences that follow from the device: AttentionInputs carries DEVICE
 * pointers (bf16, head-major [B][H][L][d], K/V with H_kv heads) instead of
 * Eigen HeadStacks, and results own device memory (DeviceBuffer, move-only)
 * instead of std::vector<Eigen::Matrix>. Results are still returned by value;
 * nothing is modified in place. Shape/config violations throw
 * std::invalid_argument("<fn>: <violations joined by '; '>") — the reference's
 * text (types.cpp:97-123, pipeline.cpp:8) — BEFORE any device work, malformed
 * masks / negative scores throw std::invalid_argument like attention.cpp:106-108
 * and selection.cpp:14-15, CUDA failures throw std::runtime_error.
 * Calls synchronize the given stream (the reference API is synchronous); the
 * allocation-free asynchronous path is the C ABI itself.
 */
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "us_api.h"

namespace unisparse_b200 {

enum class PoolStrategy { Mean = US_POOL_MEAN, Max = US_POOL_MAX, Stochastic = US_POOL_STOCHASTIC };
enum class CausalMode {
  PostSoftmaxBlockCausal = US_POST_SOFTMAX_BLOCK_CAUSAL,
  PreSoftmaxCompressedCausal = US_PRE_SOFTMAX_COMPRESSED_CAUSAL,
};
enum class SelectMode { TopP = US_SELECT_TOP_P, TopK = US_SELECT_TOP_K };

// CompressionConfig (types.hpp:54-62) + the top-k extension.
struct CompressionConfig {
  int c_q = 8;
  int c_k = 8;
  int c_h = 1;
  PoolStrategy strategy = PoolStrategy::Mean;
  double P = 0.95;
  CausalMode causal_mode = CausalMode::PostSoftmaxBlockCausal;
  std::uint64_t seed = 0;
  SelectMode select_mode = SelectMode::TopP;
  int top_k = 0;
};

// AttentionInputs (types.hpp:66-72) + batch and GQA; device pointers.
struct AttentionInputs {
  int B = 1;
  int H = 0;
  int H_kv = 0;  // 0 -> H (the reference layout)
  int L = 0;
  int d_k = 0;
  int S = 64;
  const void* Q = nullptr;  // bf16 [B][H][L][d_k] (f32 when f32 = true)
  const void* K = nullptr;  // bf16 [B][H_kv][L][d_k]
  const void* V = nullptr;  // bf16 [B][H_kv][L][d_k]
  bool f32 = false;         // Q/K/V hold f32 (the reference HeadStack<float> storage):
                            // pooled as f32 (fp64 sums); attention runs on bf16 copies
  cudaStream_t stream = nullptr;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n) check_cuda(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)), "cudaMalloc");
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  T* data() const { return p_; }
  size_t size() const { return n_; }
  std::vector<T> to_host() const {
    std::vector<T> h(n_);
    if (n_) check_cuda(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// CompressedViews (compression.hpp:79-85): f32 planes on the device.
struct CompressedViews {
  DeviceBuffer<float> Qc;  // [B][H/c_h][L/c_q][d_k]
  DeviceBuffer<float> Kc;  // [B][H/c_h][L/c_k][d_k]
  CompressionConfig cfg;
  int B = 1, H = 0, L = 0, d_k = 0;
};

// BlockMask (selection.hpp:28-37): one plane per compressed head, broadcast to
// its c_h member heads (selection.cpp:80-84). Bits [B][planes][N][ceil(N/32)].
struct BlockMask {
  int B = 1, H = 0, N = 0, W = 0, c_h = 1;
  double P_used = 0.0;
  DeviceBuffer<uint32_t> bits;
  DeviceBuffer<int32_t> counts;     // [B][planes][N]
  DeviceBuffer<double> coverage;    // [B][planes][N]
  int planes() const { return H / c_h; }
  std::int64_t selected_in_head(int h) const {  // summed over the batch
    const std::vector<int32_t> c = counts.to_host();
    std::int64_t s = 0;
    for (int b = 0; b < B; ++b)
      for (int i = 0; i < N; ++i) s += c[(size_t(b) * planes() + h / c_h) * N + i];
    return s;
  }
  std::int64_t selected_total() const {
    std::int64_t s = 0;
    for (int h = 0; h < H; ++h) s += selected_in_head(h);
    return s;
  }
};

// FlopBreakdown (metrics.hpp:16-27).
struct FlopBreakdown {
  std::uint64_t compression = 0, compressed_qk = 0, softmax_aggregation = 0, top_p = 0,
                sparse_attention = 0, dense_attention = 0;
};

// SparsityReport (metrics.hpp:77-83).
struct SparsityReport {
  std::vector<double> rho;
  double rho_mean = 0.0;
  std::vector<std::int64_t> selected;
  FlopBreakdown flops;
  BlockMask mask;
};

// AttentionOutput (attention.hpp:8-12): O bf16 (bit pattern), lse f32 natural log.
struct AttentionOutput {
  DeviceBuffer<std::uint16_t> O;  // [B][H][L][d_k]
  DeviceBuffer<float> lse;        // [B][H][L]
};

struct UniSparseResult {
  AttentionOutput out;
  SparsityReport report;
};

namespace detail {

inline us_params params(const AttentionInputs& in, const CompressionConfig& cfg, bool sync_check) {
  us_params p{};
  p.B = in.B;
  p.H = in.H;
  p.H_kv = in.H_kv ? in.H_kv : in.H;
  p.L = in.L;
  p.d_k = in.d_k;
  p.S = in.S;
  p.c_q = cfg.c_q;
  p.c_k = cfg.c_k;
  p.c_h = cfg.c_h;
  p.strategy = int32_t(cfg.strategy);
  p.causal_mode = int32_t(cfg.causal_mode);
  p.select_mode = int32_t(cfg.select_mode);
  p.P = cfg.P;
  p.top_k = cfg.top_k;
  p.flags = sync_check ? US_FLAG_SYNC_CHECK : 0;
  p.seed = cfg.seed;
  p.dtype = in.f32 ? US_DTYPE_F32 : US_DTYPE_BF16;
  return p;
}

inline void raise(us_status s) {
  if (s == US_OK) return;
  const std::string msg = us_last_error();
  switch (s) {
    case US_ERR_INVALID_ARGUMENT:
    case US_ERR_INVALID_MASK:
    case US_ERR_NONFINITE:
      throw std::invalid_argument(msg);
    case US_ERR_UNSUPPORTED:
      throw std::domain_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}

// validate_inputs (types.cpp:97-123) + GPU-path limits: throws before any device work.
inline void validate(const char* who, const us_params& p, bool need_compression = true) {
  raise(us_check_params(&p, who, need_compression ? 1 : 0));
}

inline DeviceBuffer<uint8_t> workspace(const us_params& p) {
  return DeviceBuffer<uint8_t>(us_workspace_bytes(&p) + 256);
}
// the attention entry points' (much smaller) workspace
inline DeviceBuffer<uint8_t> attention_workspace(const us_params& p) {
  return DeviceBuffer<uint8_t>(us_attention_workspace_bytes(&p) + 256);
}

inline FlopBreakdown flops(const us_params& p) {
  uint64_t f[6];
  raise(us_selection_flops(&p, US_PROXY_UNISPARSE, 8, f));
  FlopBreakdown r;
  r.compression = f[0];
  r.compressed_qk = f[1];
  r.softmax_aggregation = f[2];
  r.top_p = f[3];
  r.dense_attention = f[5];
  return r;
}

inline BlockMask alloc_mask(const us_params& p) {
  BlockMask m;
  m.B = p.B;
  m.H = p.H;
  m.N = p.L / p.S;
  m.W = (m.N + 31) / 32;
  m.c_h = p.c_h;
  m.P_used = p.P;
  const size_t rows = size_t(p.B) * (p.H / p.c_h) * m.N;
  m.bits = DeviceBuffer<uint32_t>(rows * m.W);
  m.counts = DeviceBuffer<int32_t>(rows);
  m.coverage = DeviceBuffer<double>(rows);
  return m;
}

// make_sparsity_report (metrics.cpp:226-237).
inline SparsityReport report(const us_params& p, BlockMask&& mask) {
  SparsityReport r;
  const double causal = double(mask.N) * (mask.N + 1) / 2.0 * p.B;
  r.flops = flops(p);
  std::int64_t total = 0;
  for (int h = 0; h < p.H; ++h) {
    const std::int64_t s = mask.selected_in_head(h);
    r.selected.push_back(s);
    r.rho.push_back(1.0 - double(s) / causal);
    total += s;
  }
  double acc = 0.0;
  for (double x : r.rho) acc += x;
  r.rho_mean = r.rho.empty() ? 0.0 : acc / double(r.rho.size());
  r.flops.sparse_attention = std::uint64_t(total) * 4ull * p.S * p.S * p.d_k;
  r.mask = std::move(mask);
  return r;
}

}  // namespace detail

inline CompressedViews compress(const AttentionInputs& in, const CompressionConfig& cfg) {
  const us_params p = detail::params(in, cfg, true);
  detail::validate("compress", p);
  CompressedViews v;
  v.cfg = cfg;
  v.B = in.B;
  v.H = in.H;
  v.L = in.L;
  v.d_k = in.d_k;
  const size_t planes = size_t(in.B) * (in.H / cfg.c_h);
  v.Qc = DeviceBuffer<float>(planes * (in.L / cfg.c_q) * in.d_k);
  v.Kc = DeviceBuffer<float>(planes * (in.L / cfg.c_k) * in.d_k);
  DeviceBuffer<std::uint8_t> ws;  // d_k outside {64, 128}: zero-padded copies in the workspace
  if (in.d_k != 64 && in.d_k != 128) ws = detail::workspace(p);
  detail::raise(us_compress(&p, in.Q, in.K, v.Qc.data(), v.Kc.data(), ws.data(), ws.size(), in.stream));
  return v;
}

enum class ProxyTag { UniSparse = US_PROXY_UNISPARSE, Antidiagonal = US_PROXY_ANTIDIAGONAL,
                      LastBlockProbe = US_PROXY_LAST_BLOCK };

// select_blocks(proxy, in, cfg, stride) (pipeline.hpp:19-20): the competitor proxies
// score per original head (c_h forced to 1, pipeline.cpp:11).
inline SparsityReport select_blocks(ProxyTag proxy, const AttentionInputs& in, const CompressionConfig& cfg,
                                    int stride = 8) {
  CompressionConfig c = cfg;
  if (proxy != ProxyTag::UniSparse) c.c_h = 1;
  const us_params p = detail::params(in, c, true);
  detail::validate("select_blocks", p, proxy == ProxyTag::UniSparse);
  BlockMask m = detail::alloc_mask(p);
  DeviceBuffer<uint8_t> ws(us_proxy_workspace_bytes(&p, int32_t(proxy), stride) + 256);
  us_selection sel{m.bits.data(), m.counts.data(), m.coverage.data(), nullptr, nullptr};
  detail::raise(us_select_proxy(&p, int32_t(proxy), stride, in.Q, in.K, &sel, ws.data(), ws.size(), in.stream));
  SparsityReport r = detail::report(p, std::move(m));
  uint64_t f[6];
  detail::raise(us_selection_flops(&p, int32_t(proxy), stride, f));
  r.flops.compression = f[0];
  r.flops.compressed_qk = f[1];
  r.flops.softmax_aggregation = f[2];
  r.flops.top_p = f[3];
  return r;
}

inline SparsityReport select_blocks(const AttentionInputs& in, const CompressionConfig& cfg) {
  const us_params p = detail::params(in, cfg, true);
  detail::validate("select_blocks", p);
  BlockMask m = detail::alloc_mask(p);
  auto ws = detail::workspace(p);
  us_selection sel{m.bits.data(), m.counts.data(), m.coverage.data(), nullptr, nullptr};
  detail::raise(us_select(&p, in.Q, in.K, &sel, ws.data(), ws.size(), in.stream));
  return detail::report(p, std::move(m));
}

// scores: device f32 [B][H/c_h][N][N] (j <= i read); H = original head count.
inline BlockMask build_block_mask(const float* scores, int B, int H, int N, const CompressionConfig& cfg,
                                  cudaStream_t stream = nullptr) {
  AttentionInputs in;
  in.B = B;
  in.H = H;
  in.L = N * 64;
  in.d_k = 64;
  us_params p = detail::params(in, cfg, true);
  if (cfg.c_h <= 0 || H % cfg.c_h != 0)
    throw std::invalid_argument("build_block_mask: H=" + std::to_string(H) + " not divisible by c_h=" +
                                std::to_string(cfg.c_h));
  BlockMask m = detail::alloc_mask(p);
  auto ws = detail::workspace(p);
  us_selection sel{m.bits.data(), m.counts.data(), m.coverage.data(), nullptr, nullptr};
  detail::raise(us_build_block_mask(&p, scores, &sel, ws.data(), ws.size(), stream));
  return m;
}

inline AttentionOutput block_sparse_attention(const AttentionInputs& in, const BlockMask& mask) {
  CompressionConfig c1;
  c1.c_q = c1.c_k = c1.c_h = 1;
  const us_params p = detail::params(in, c1, true);
  detail::validate("block_sparse_attention", p, false);
  if (mask.N != in.L / in.S || mask.B != in.B || mask.H != in.H)
    throw std::invalid_argument("block_sparse_attention: mask shape does not match the inputs");
  AttentionOutput out;
  out.O = DeviceBuffer<std::uint16_t>(size_t(in.B) * in.H * in.L * in.d_k);
  out.lse = DeviceBuffer<float>(size_t(in.B) * in.H * in.L);
  auto ws = detail::attention_workspace(p);
  detail::raise(us_sparse_attention(&p, in.Q, in.K, in.V, mask.bits.data(), mask.c_h, out.O.data(),
                                    out.lse.data(), ws.data(), ws.size(), in.stream));
  return out;
}

inline UniSparseResult unisparse_attn(const AttentionInputs& in, const CompressionConfig& cfg) {
  const us_params p = detail::params(in, cfg, true);
  detail::validate("select_blocks", p);  // pipeline.cpp:19-24 validates via select_blocks
  BlockMask m = detail::alloc_mask(p);
  UniSparseResult r;
  r.out.O = DeviceBuffer<std::uint16_t>(size_t(in.B) * in.H * in.L * in.d_k);
  r.out.lse = DeviceBuffer<float>(size_t(in.B) * in.H * in.L);
  auto ws = detail::workspace(p);
  us_selection sel{m.bits.data(), m.counts.data(), m.coverage.data(), nullptr, nullptr};
  detail::raise(us_unisparse_attention(&p, in.Q, in.K, in.V, r.out.O.data(), r.out.lse.data(), &sel,
                                       ws.data(), ws.size(), in.stream));
  r.report = detail::report(p, std::move(m));
  return r;
}

inline AttentionOutput dense_attention(const AttentionInputs& in, bool causal = true) {
  CompressionConfig c1;
  c1.c_q = c1.c_k = c1.c_h = 1;
  us_params p = detail::params(in, c1, true);
  if (!causal) p.flags |= US_FLAG_NONCAUSAL;
  detail::validate("dense_attention", p, false);
  AttentionOutput out;
  out.O = DeviceBuffer<std::uint16_t>(size_t(in.B) * in.H * in.L * in.d_k);
  out.lse = DeviceBuffer<float>(size_t(in.B) * in.H * in.L);
  DeviceBuffer<std::uint8_t> ws;  // f32 inputs: bf16 copies; d_k outside {64, 128}: padded copies
  if (in.f32 || (in.d_k != 64 && in.d_k != 128)) ws = detail::attention_workspace(p);
  detail::raise(us_dense_attention(&p, in.Q, in.K, in.V, out.O.data(), out.lse.data(), ws.data(), ws.size(),
                                   in.stream));
  return out;
}

// selection_flops (metrics.cpp:44-81) for the UniSparse proxy.
inline FlopBreakdown selection_flops(int L, int H, int d_k, int S, const CompressionConfig& cfg) {
  AttentionInputs in;
  in.H = H;
  in.L = L;
  in.d_k = d_k;
  in.S = S;
  return detail::flops(detail::params(in, cfg, false));
}

}  // namespace unisparse_b200
