// api.cu — the C ABI (include/us_api.h): validation with the reference's
// messages, workspace layout, TMA descriptors and kernel orchestration.
//
// Pipeline of us_unisparse_attention (pipeline.cpp:19-24), all on one stream:
//   compress Q, compress K (f32 + per-plane absmax)        compress.cu
//   split Q, split K (fp16 hi/lo, per-plane 2^e)           compress.cu
//   proxy pass 1 (row lse), pass 2 (block scores)          proxy.cu   (tcgen05)
//   select (+ exact fallback for uncertified rows)         select.cu
//   block-sparse attention                                 attention.cu (tcgen05)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host_util.hpp"
#include "kernels.cuh"

namespace us {

namespace {
thread_local std::string g_err;
thread_local int g_launches = 0;

// stage-boundary events: slot c uses events [5c, 5c+5)
struct Profiler {
  std::vector<cudaEvent_t> ev;
  int max_calls = 0, next = 0;
  bool on() const { return max_calls > 0; }
  void mark(int call, int k, cudaStream_t st) {
    if (call >= 0 && call < max_calls) cudaEventRecord(ev[size_t(call) * 5 + k], st);
  }
};
thread_local Profiler g_prof;
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
int& launch_counter() { return g_launches; }

namespace {

constexpr int kGpuBlock = 64;

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

struct Checked {
  std::vector<std::string> errors;       // reference validate_inputs violations
  std::vector<std::string> unsupported;  // valid for the reference, not on this GPU path
};

// validate_inputs (types.cpp:97-123) — same order and text — then GQA/batch
// extensions, then GPU-path constraints.
Checked check(const us_params& p, bool need_compression) {
  Checked c;
  auto& e = c.errors;
  if (p.H <= 0) e.push_back("H must be positive");
  if (p.L <= 0) e.push_back("L must be positive");
  if (p.d_k <= 0) e.push_back("d_k must be positive");
  if (p.S <= 0) e.push_back("S must be positive");
  if (p.L > 0 && p.S > 0 && p.L % p.S != 0)
    e.push_back("L=" + std::to_string(p.L) + " not divisible by S=" + std::to_string(p.S));
  if (p.c_q <= 0) e.push_back("c_q must be positive");
  if (p.c_k <= 0) e.push_back("c_k must be positive");
  if (p.c_h <= 0) e.push_back("c_h must be positive");
  if (p.S > 0 && p.c_q > 0 && p.S % p.c_q != 0)
    e.push_back("S=" + std::to_string(p.S) + " not divisible by c_q=" + std::to_string(p.c_q));
  if (p.S > 0 && p.c_k > 0 && p.S % p.c_k != 0)
    e.push_back("S=" + std::to_string(p.S) + " not divisible by c_k=" + std::to_string(p.c_k));
  if (p.H > 0 && p.c_h > 0 && p.H % p.c_h != 0)
    e.push_back("H=" + std::to_string(p.H) + " not divisible by c_h=" + std::to_string(p.c_h));
  if (!(p.P > 0.0) || p.P > 1.0) e.push_back("P must lie in (0, 1]");
  if (p.H_kv <= 0) e.push_back("H_kv must be positive");
  if (p.H > 0 && p.H_kv > 0 && p.H % p.H_kv != 0)
    e.push_back("H=" + std::to_string(p.H) + " not divisible by H_kv=" + std::to_string(p.H_kv));
  if (p.B <= 0) e.push_back("B must be positive");
  if (p.head0 < 0) e.push_back("head0 must be non-negative");
  if (p.dtype != US_DTYPE_BF16 && p.dtype != US_DTYPE_F32) e.push_back("unknown dtype");
  if (p.select_mode != US_SELECT_TOP_P && p.select_mode != US_SELECT_TOP_K)
    e.push_back("unknown select_mode");
  if (p.select_mode == US_SELECT_TOP_K && p.top_k < 1) e.push_back("top_k must be positive");
  if (p.causal_mode != US_POST_SOFTMAX_BLOCK_CAUSAL && p.causal_mode != US_PRE_SOFTMAX_COMPRESSED_CAUSAL)
    e.push_back("unknown causal_mode");
  if (!e.empty()) return c;
  auto& u = c.unsupported;
  if (p.d_k > 128)
    u.push_back("d_k=" + std::to_string(p.d_k) + " unsupported on the GPU path (at most 128)");
  if (p.S != kGpuBlock && p.S != 2 * kGpuBlock && p.S != 4 * kGpuBlock)
    u.push_back("S=" + std::to_string(p.S) + " unsupported on the GPU path (64, 128 or 256)");
  if (p.L / kGpuBlock > 4096) u.push_back("L/64 above 4096 unsupported on the GPU path");
  if ((long long)p.B * p.H * p.L >= (1ll << 31)) u.push_back("B*H*L must stay below 2^31 rows");
  if (need_compression) {
    if (p.strategy != US_POOL_MEAN && p.strategy != US_POOL_MAX && p.strategy != US_POOL_STOCHASTIC)
      u.push_back("unknown pooling strategy");
    if (!is_pow2(p.S / p.c_q) || !is_pow2(p.S / p.c_k))
      u.push_back("S/c_q and S/c_k must be powers of two on the GPU path");
  }
  return c;
}

std::string joined(const std::vector<std::string>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "; " : "") + v[i];
  return s;
}

us_status gate(const us_params* p, const char* who, bool need_compression) {
  g_launches = 0;
  if (!p) {
    set_error(std::string(who) + ": null params");
    return US_ERR_INVALID_ARGUMENT;
  }
  Checked c = check(*p, need_compression);
  if (!c.errors.empty()) {
    set_error(std::string(who) + ": " + joined(c.errors));
    return US_ERR_INVALID_ARGUMENT;
  }
  if (!c.unsupported.empty()) {
    set_error(std::string(who) + ": " + joined(c.unsupported));
    return US_ERR_UNSUPPORTED;
  }
  return US_OK;
}

// ---------------------------------------------------------------- geometry
// d_k outside {64, 128} (the reference accepts any d_k, types.hpp:66-72): the entry points
// stage copies zero-padded to the next supported width in the workspace and run the same
// kernels at that width (zeros pool to exact zeros and add exact zeros to every dot product,
// so compressed rows, logits, masks and outputs equal the unpadded computation); the
// softmax scale keeps the caller's d_k, set for the duration of the inner call here.
thread_local int t_scale_dk = 0;
struct ScaleDk {
  int prev;
  explicit ScaleDk(int d) : prev(t_scale_dk) { t_scale_dk = d; }
  ~ScaleDk() { t_scale_dk = prev; }
};
int padded_dk(int d) { return d <= 64 ? 64 : 128; }
bool needs_pad(const us_params& p) { return p.d_k != padded_dk(p.d_k); }

struct Geo {
  int B, H, H_kv, G, L, D, Ds, S, N, W, Hc, Lq, Lk, rq, rk;
  bool kv_dedup;
  int kv_planes, kv_mul, kv_div;
  explicit Geo(const us_params& p) {
    B = p.B;
    H = p.H;
    H_kv = p.H_kv;
    G = H / H_kv;
    L = p.L;
    D = p.d_k;
    Ds = t_scale_dk > 0 ? t_scale_dk : p.d_k;  // d_k of the softmax scale 1/sqrt(d_k)
    S = p.S;
    N = L / S;
    W = (N + 31) / 32;
    Hc = H / p.c_h;
    Lq = L / p.c_q;
    Lk = L / p.c_k;
    rq = S / p.c_q;
    rk = S / p.c_k;
    // one pooled K per KV head when the expanded copies are identical: every strategy
    // but stochastic (whose per-head seeds differ, compression.cpp:19-20)
    kv_dedup = (G % p.c_h) == 0 && p.strategy != US_POOL_STOCHASTIC;
    kv_planes = kv_dedup ? H_kv : Hc;
    kv_mul = kv_dedup ? p.c_h : 1;
    kv_div = kv_dedup ? G : 1;
  }
};

struct Ws {
  size_t err, first_bad, fb_count, absmax_q, absmax_k, exp_q, exp_k, fb_rows, qc, kc, qh, ql, kh,
      kl, lse2, part, tmax, scores, mask, conv, mask64, items, total;
  size_t header_bytes;  // [0, header_bytes) is cleared before each selection
};

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// scores_region: the [B][planes][N][N] f32 block-score tensor, needed only by the
// competitor proxies and exact_block_mass; the UniSparse path fuses the block
// scores into the selection (select_fused_kernel) and never materialises them.
// attn_only: the attention entry points (block_sparse_attention, dense_attention) need
// only the error header, the bf16 copies of f32 inputs, the 64-granular mask and the
// attention64 item table — not the proxy / selection buffers, which at c = 1 (the
// attention-only params) would scale with the uncompressed length.
Ws layout(const us_params& p, bool scores_region = false, bool attn_only = false) {
  Geo g(p);
  Ws w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = al(o + bytes);
    return at;
  };
  const size_t qplanes = size_t(g.B) * g.Hc, kplanes = size_t(g.B) * g.kv_planes;
  w.err = take(4);
  w.first_bad = take(4);
  w.fb_count = take(4);
  w.absmax_q = take(4 * qplanes);
  w.absmax_k = take(4 * kplanes);
  w.header_bytes = o;
  if (!attn_only) {
  w.exp_q = take(4 * qplanes * g.Lq);  // one scale exponent per composite query row
  w.exp_k = take(4 * kplanes);
  const size_t rows = qplanes * g.N;
  w.fb_rows = take(4 * rows);
  // +128 rows of padding keep every TMA box inside the allocation
  const size_t qrows = qplanes * g.Lq + 128, krows = kplanes * g.Lk + 128;
  w.qc = 0;  // (Q is pooled straight into its fp16 hi/lo pair: no f32 copy in the workspace)
  w.kc = take(4 * krows * g.D);
  w.qh = take(2 * qrows * g.D);
  w.ql = take(2 * qrows * g.D);
  w.kh = take(2 * krows * g.D);
  w.kl = take(2 * krows * g.D);
  w.lse2 = take(4 * qplanes * g.Lq);
  // slot partials of the one-pass proxy: [qplanes][T][Lq][128/sw] (= Lq * Lk/sw per plane)
  const size_t T = (size_t(g.Lk) + 127) / 128;
  const size_t ns = 128 / size_t(proxy_slot_width(g.rk));
  w.part = take(4 * qplanes * T * g.Lq * ns);
  w.tmax = take(4 * qplanes * T * g.Lq);
  w.scores = scores_region ? take(4 * rows * g.N) : 0;
  w.mask = take(4 * rows * g.W);
  }
  // f32 inputs: bf16 copies of Q, K, V for the attention kernels
  w.conv = p.dtype == US_DTYPE_F32 ? take(2 * (size_t(g.B) * g.H + 2 * size_t(g.B) * g.H_kv) * g.L * g.D) : 0;
  // S > 64: the 64-granular copy of the block mask the attention kernels walk (one plane per head)
  const size_t n64 = size_t(g.L) / kGpuBlock;
  w.mask64 = g.S != kGpuBlock ? take(4 * size_t(g.B) * g.H * n64 * ((n64 + 31) / 32)) : 0;
  // attention64.cu work-item table (groups sorted by selected-block count)
  w.items = take(attention64_ws_bytes(g.B, g.H, g.H_kv, int(n64)));
  w.total = o;
  return w;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + off);
}

us_status need_ws(const us_params& p, void* ws, size_t bytes, const char* who, bool scores_region = false,
                  bool attn_only = false) {
  const size_t need = layout(p, scores_region, attn_only).total;
  if (!ws || bytes < need) {
    set_error(std::string(who) + ": workspace of " + std::to_string(need) + " bytes required");
    return US_ERR_WORKSPACE;
  }
  return US_OK;
}

// Padded d_k staging (see padded_dk): the inner call's workspace comes first (so the error
// header sits where us_check_device_errors looks for it), then zero-padded copies of the
// inputs and of the outputs the call produces at the padded width.
struct PadWs {
  size_t q, k, v, o, qc, kc, total;
};
PadWs pad_layout(const us_params& p) {
  Geo g(p);
  const size_t Dp = size_t(padded_dk(p.d_k)), es = p.dtype == US_DTYPE_F32 ? 4 : 2;
  PadWs w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = al(o + bytes);
    return at;
  };
  w.q = take(es * size_t(g.B) * g.H * g.L * Dp);
  w.k = take(es * size_t(g.B) * g.H_kv * g.L * Dp);
  w.v = take(es * size_t(g.B) * g.H_kv * g.L * Dp);
  w.o = take(2 * size_t(g.B) * g.H * g.L * Dp);
  w.qc = take(4 * size_t(g.B) * g.Hc * g.Lq * Dp);
  w.kc = take(4 * size_t(g.B) * g.Hc * g.Lk * Dp);
  w.total = o;
  return w;
}
us_params padded_params(const us_params& p) {
  us_params q = p;
  q.d_k = padded_dk(p.d_k);
  return q;
}
size_t padded_ws_bytes(const us_params& p, bool attn_only = false) {
  return al(layout(padded_params(p), false, attn_only).total) + pad_layout(p).total;
}

struct PadStage {
  us_params pp;        // the same call at the padded width
  size_t inner_bytes;  // workspace of the inner call, at the start of the caller's
  uint8_t* base;       // padded copies
  PadWs w;
  size_t es;           // bytes per input element
};
// inner_total: the inner call's workspace at the padded width (default: layout(pp))
us_status pad_begin(const us_params& p, void* ws, size_t bytes, const char* who, PadStage& ps,
                    size_t inner_total = 0) {
  ps.pp = padded_params(p);
  ps.inner_bytes = al(inner_total ? inner_total : layout(ps.pp).total);
  ps.w = pad_layout(p);
  ps.es = p.dtype == US_DTYPE_F32 ? 4 : 2;
  const size_t need = ps.inner_bytes + ps.w.total;
  if (!ws || bytes < need) {
    set_error(std::string(who) + ": workspace of " + std::to_string(need) + " bytes required (d_k=" +
              std::to_string(p.d_k) + " runs zero-padded to " + std::to_string(ps.pp.d_k) + ")");
    return US_ERR_WORKSPACE;
  }
  ps.base = static_cast<uint8_t*>(ws) + ps.inner_bytes;
  return US_OK;
}
// rows x d -> rows x Dp with zero columns [d, Dp)
us_status pad_rows(const void* src, void* dst, size_t rows, int d, int Dp, size_t es, cudaStream_t st) {
  US_CUDA_TRY(cudaMemcpy2DAsync(dst, Dp * es, src, d * es, d * es, rows, cudaMemcpyDeviceToDevice, st), "d_k pad copy");
  US_CUDA_TRY(cudaMemset2DAsync(static_cast<uint8_t*>(dst) + d * es, Dp * es, 0, (Dp - d) * es, rows, st),
              "d_k pad clear");
  return US_OK;
}
us_status unpad_rows(const void* src, void* dst, size_t rows, int d, int Dp, size_t es, cudaStream_t st) {
  US_CUDA_TRY(cudaMemcpy2DAsync(dst, d * es, src, Dp * es, d * es, rows, cudaMemcpyDeviceToDevice, st), "d_k unpad copy");
  return US_OK;
}
// stage Q (and K, V when given) at the padded width
us_status pad_inputs(const us_params& p, const PadStage& ps, const void* Q, const void* K, const void* V,
                     cudaStream_t st) {
  Geo g(p);
  us_status s;
  const int Dp = ps.pp.d_k;
  if (Q && (s = pad_rows(Q, ps.base + ps.w.q, size_t(g.B) * g.H * g.L, g.D, Dp, ps.es, st)) != US_OK) return s;
  if (K && (s = pad_rows(K, ps.base + ps.w.k, size_t(g.B) * g.H_kv * g.L, g.D, Dp, ps.es, st)) != US_OK) return s;
  if (V && (s = pad_rows(V, ps.base + ps.w.v, size_t(g.B) * g.H_kv * g.L, g.D, Dp, ps.es, st)) != US_OK) return s;
  return US_OK;
}

// compress + split + proxy (logits, row LSE, slot partials). The block scores are
// formed by the fused selection (launch_select_fused with *pa_out).
us_status run_proxy(const us_params& p, const void* Q, const void* K, void* ws, cudaStream_t st,
                    ProxyArgs* pa_out, int prof_call = -1) {
  Geo g(p);
  Ws w = layout(p);
  US_CUDA_TRY(cudaMemsetAsync(ws, 0, w.header_bytes, st), "workspace clear");
  // Q: pooling fused with the fp16 hi/lo split at a per-row power-of-two scale
  // (compress.cu); K: f32 + per-plane |max|, then the split (K is 4-8x smaller)
  CompressArgs cq{static_cast<const uint16_t*>(Q), g.B, g.H, g.L, g.D, p.c_q, g.Hc, p.c_h, 1,
                  nullptr, nullptr, p.strategy, 0, p.seed, p.head0,
                  at<__half>(ws, w.qh), at<__half>(ws, w.ql), at<int>(ws, w.exp_q), p.dtype == US_DTYPE_F32};
  us_status s = launch_compress(cq, st);
  if (s != US_OK) return s;
  CompressArgs ck{static_cast<const uint16_t*>(K), g.B, g.H_kv, g.L, g.D, p.c_k, g.kv_planes,
                  g.kv_dedup ? 1 : p.c_h, g.kv_dedup ? 1 : g.G, at<float>(ws, w.kc),
                  at<uint32_t>(ws, w.absmax_k), p.strategy, 1, p.seed, p.head0,
                  nullptr, nullptr, nullptr, p.dtype == US_DTYPE_F32};
  if ((s = launch_compress(ck, st)) != US_OK) return s;
  SplitArgs sk{at<float>(ws, w.kc), g.B * g.kv_planes, g.Lk, g.D, at<uint32_t>(ws, w.absmax_k),
               at<int>(ws, w.exp_k), at<__half>(ws, w.kh), at<__half>(ws, w.kl)};
  if ((s = launch_split(sk, st)) != US_OK) return s;

  g_prof.mark(prof_call, 1, st);
  const uint64_t krows = uint64_t(g.B) * g.kv_planes * g.Lk + 128;
  CUtensorMap tKh, tKl;
  if ((s = make_tmap_2d_16b(&tKh, at<void>(ws, w.kh), krows, g.D, 128, 64, false)) != US_OK) return s;
  if ((s = make_tmap_2d_16b(&tKl, at<void>(ws, w.kl), krows, g.D, 128, 64, false)) != US_OK) return s;
  ProxyArgs pa{};
  pa.B = g.B;
  pa.Hc = g.Hc;
  pa.Lq = g.Lq;
  pa.Lk = g.Lk;
  pa.N = g.N;
  pa.D = g.D;
  pa.rq = g.rq;
  pa.rk = g.rk;
  pa.c_q = p.c_q;
  pa.c_k = p.c_k;
  pa.causal_mode = p.causal_mode;
  pa.kv_planes = g.kv_planes;
  pa.kv_mul = g.kv_mul;
  pa.kv_div = g.kv_div;
  pa.exp_q = at<int>(ws, w.exp_q);
  pa.q_row_exp = 1;
  pa.exp_k = at<int>(ws, w.exp_k);
  pa.qh = at<__half>(ws, w.qh);
  pa.ql = at<__half>(ws, w.ql);
  pa.T = (g.Lk + 127) / 128;
  pa.sw = proxy_slot_width(g.rk);
  pa.part = at<float>(ws, w.part);
  pa.tmax = at<float>(ws, w.tmax);
  pa.lse2 = at<float>(ws, w.lse2);
  pa.scores = nullptr;
  pa.scale_log2 = float(1.4426950408889634 / std::sqrt(double(g.Ds)));
  pa.x3 = 1;
  pa.finalize = 0;
  *pa_out = pa;
  return launch_proxy(pa, tKh, tKl, st);
}

// params whose workspace layout fits the antidiagonal proxy: composite rows of one
// phase class are L / stride long, like a compression factor of `stride`
us_params antidiag_params(const us_params& p, int stride) {
  us_params q = p;
  q.c_q = q.c_k = stride;
  q.c_h = 1;
  q.causal_mode = US_PRE_SOFTMAX_COMPRESSED_CAUSAL;
  return q;
}

// antidiagonal_block_scores (baselines.cpp:10-52) into ws.scores [B][H][N][N]: one
// pass of the proxy kernel per query phase class a (queries t = stride*t' + a sample
// the keys s = stride*s' + res, res = stride - 1 - a, s <= t), bf16 single-MMA logits
// (exact products), softmax over the sampled causal keys, region sums accumulated
// over the classes in a fixed order.
us_status run_antidiagonal(const us_params& p, int stride, const void* Q, const void* K, void* ws,
                           cudaStream_t st) {
  const us_params q = antidiag_params(p, stride);
  Geo g(q);
  Ws w = layout(q, true);
  const int Lc = g.L / stride;
  CUtensorMap tK;
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return US_ERR_CUDA;
  }
  {
    // K as (d, stride, B*H_kv*L/stride): box (64, 1, 128) = 128 keys of one phase class
    cuuint64_t dims[3] = {cuuint64_t(g.D), cuuint64_t(stride), cuuint64_t(g.B) * g.H_kv * Lc};
    cuuint64_t strides[2] = {cuuint64_t(g.D) * 2, cuuint64_t(g.D) * 2 * stride};
    cuuint32_t box[3] = {64, 1, 128};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(&tK, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(K), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (3-D K) failed (" + std::to_string(int(r)) + ")");
      return US_ERR_CUDA;
    }
  }
  ProxyArgs pa{};
  pa.B = g.B;
  pa.Hc = g.H;
  pa.Lq = Lc;
  pa.Lk = Lc;
  pa.N = g.N;
  pa.D = g.D;
  pa.rq = g.S / stride;
  pa.rk = g.S / stride;
  pa.c_q = stride;
  pa.c_k = stride;
  pa.causal_mode = US_PRE_SOFTMAX_COMPRESSED_CAUSAL;
  pa.kv_planes = g.H_kv;
  pa.kv_mul = 1;
  pa.kv_div = g.G;
  pa.T = (Lc + 127) / 128;
  pa.sw = proxy_slot_width(pa.rk);
  pa.part = at<float>(ws, w.part);
  pa.tmax = at<float>(ws, w.tmax);
  pa.lse2 = at<float>(ws, w.lse2);
  pa.scores = at<float>(ws, w.scores);
  pa.finalize = 1;
  pa.scale_log2 = float(1.4426950408889634 / std::sqrt(double(g.Ds)));
  pa.x3 = 0;
  pa.qraw = static_cast<const uint16_t*>(Q);
  pa.L = g.L;
  pa.q_row0 = 0;
  pa.q_stride = stride;
  for (int cls = 0; cls < stride; ++cls) {
    const int res = stride - 1 - cls;
    pa.q_phase = cls;
    pa.k_phase = res;
    pa.live_bias = cls >= res ? 1 : 0;
    pa.accumulate = cls > 0;
    us_status s = launch_proxy(pa, tK, tK, st);
    if (s != US_OK) return s;
  }
  return US_OK;
}

us_status run_select_rows(const us_params& p, const float* scores, int planes, uint32_t* mask,
                          const us_selection* sel, void* ws, cudaStream_t st) {
  Geo g(p);
  Ws w = layout(p);
  SelectArgs sa{};
  sa.scores = scores;
  sa.rows = g.B * planes * g.N;
  sa.N = g.N;
  sa.W = g.W;
  sa.select_mode = p.select_mode;
  sa.P = p.P;
  sa.top_k = p.top_k;
  sa.mask_bits = mask;
  sa.counts = sel ? sel->counts : nullptr;
  sa.coverage = sel ? sel->coverage : nullptr;
  sa.indices = sel ? sel->indices : nullptr;
  sa.err = at<uint32_t>(ws, w.err);
  sa.fb_count = at<int32_t>(ws, w.fb_count);
  sa.fb_rows = at<int32_t>(ws, w.fb_rows);
  return launch_select(sa, st);
}

// Fused finalize + selection on the proxy's slot partials (the UniSparse path).
us_status run_select_fused(const us_params& p, const ProxyArgs& pa, uint32_t* mask, const us_selection* sel, void* ws,
                           cudaStream_t st) {
  Geo g(p);
  Ws w = layout(p);
  SelectArgs sa{};
  sa.scores_out = sel ? sel->scores : nullptr;  // raw block scores only when asked for
  sa.rows = g.B * g.Hc * g.N;
  sa.N = g.N;
  sa.W = g.W;
  sa.select_mode = p.select_mode;
  sa.P = p.P;
  sa.top_k = p.top_k;
  sa.mask_bits = mask;
  sa.counts = sel ? sel->counts : nullptr;
  sa.coverage = sel ? sel->coverage : nullptr;
  sa.indices = sel ? sel->indices : nullptr;
  sa.err = at<uint32_t>(ws, w.err);
  sa.fb_count = at<int32_t>(ws, w.fb_count);
  sa.fb_rows = at<int32_t>(ws, w.fb_rows);
  return launch_select_fused(pa, sa, st);
}

// Attention kernel selection (calibration knob, US_ATTN_IMPL): 0 = automatic
// (default: masks with the item-table workspace launch both attention64.cu and
// attention.cu, the device-side density gate attn::m64_wins running one of them; dense
// and workspace-less calls run attention.cu), 1 = attention.cu (two M=128 query tiles
// per CTA, 64-key steps), 2 = attention2.cu, 3 = attention.cu with one tile per CTA,
// 4 = attention_kt.cu whenever d_k = 128, 5 = attention_tp.cu (decoupled softmax),
// 6 = attention64.cu for every mask (M = 64 chains). 2-5: calibration build only.
std::atomic<int> g_attn_impl{-1};
int attention_impl() {
  int v = g_attn_impl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("US_ATTN_IMPL");
    v = (e && std::atoi(e) >= 1 && std::atoi(e) <= 6) ? std::atoi(e) : 0;
    g_attn_impl.store(v, std::memory_order_relaxed);
  }
  return v;
}

// Calibration knob: US_ATTN_PAIRING=0 keeps the fixed (01|23) tile pairing.
std::atomic<int> g_attn_pairing{-1};
int attention_pairing() {
  int v = g_attn_pairing.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("US_ATTN_PAIRING");
    v = (e && std::atoi(e) == 0) ? 0 : 1;
    g_attn_pairing.store(v, std::memory_order_relaxed);
  }
  return v;
}

// The attention kernels: bf16 Q/K/V, 64-granular masks (p.S == 64, p.dtype == bf16).
us_status run_attention_core(const us_params& p, const void* Q, const void* K, const void* V,
                             const uint32_t* mask, int hpp, void* O, float* lse, cudaStream_t st, uint32_t* err,
                             int32_t* first_bad, int32_t* items) {
  Geo g(p);
  us_status s;
  CUtensorMap tQ, tK, tV;
  if ((s = make_tmap_2d_16b(&tQ, Q, uint64_t(g.B) * g.H * g.L, g.D, 64, 64, true)) != US_OK) return s;
  if ((s = make_tmap_2d_16b(&tK, K, uint64_t(g.B) * g.H_kv * g.L, g.D, 64, 64, true)) != US_OK) return s;
  if ((s = make_tmap_2d_16b(&tV, V, uint64_t(g.B) * g.H_kv * g.L, g.D, 64, 64, true)) != US_OK) return s;
  CUtensorMap tK3, tV3;  // attention.cu: one TMA per K / V tile (all d-chunks)
  if ((s = make_tmap_rows_chunked(&tK3, K, uint64_t(g.B) * g.H_kv * g.L, g.D, 64)) != US_OK) return s;
  if ((s = make_tmap_rows_chunked(&tV3, V, uint64_t(g.B) * g.H_kv * g.L, g.D, 64)) != US_OK) return s;
  AttnArgs a{};
  a.B = g.B;
  a.H = g.H;
  a.H_kv = g.H_kv;
  a.L = g.L;
  a.N = g.N;
  a.W = g.W;
  a.D = g.D;
  a.group_mode = (g.G % 4 == 0) ? 0 : (g.G == 2 ? 1 : 2);
  a.pairing = attention_pairing();
  a.heads_per_plane = hpp;
  a.planes = g.H / hpp;
  a.mask = mask;
  a.Q = static_cast<const __nv_bfloat16*>(Q);
  a.O = static_cast<__nv_bfloat16*>(O);
  a.lse = lse;
  a.scale_log2 = float(1.4426950408889634 / std::sqrt(double(g.Ds)));
  a.noncausal = (!mask && (p.flags & US_FLAG_NONCAUSAL)) ? 1 : 0;
  a.err = err;
  a.first_bad = first_bad;
  const int impl = attention_impl();
#ifdef US_CALIBRATION
  // calibration variants (libunisparse_b200_calib.so only; measured slower, DESIGN.md §3 a6)
  if (g.D == 128 && impl == 4 && !a.noncausal) {
    CUtensorMap tQ3;
    if ((s = make_tmap_rows_chunked(&tQ3, Q, uint64_t(g.B) * g.H * g.L, g.D, 64)) != US_OK) return s;
    return launch_attention_kt(a, tQ3, tK, tV3, st);
  }
  if (impl == 2 && !a.noncausal) return launch_attention2(a, tK, tV, st);
  a.one_tile = impl == 3 ? 1 : 0;
  if (impl == 5) return launch_attention_tp(a, tQ, tK3, tV3, st);
#endif
  CUtensorMap tQa;  // attention64.cu: one TMA per 64 Q rows (all d-chunks)
  if (mask && (s = make_tmap_rows_chunked(&tQa, Q, uint64_t(g.B) * g.H * g.L, g.D, 64)) != US_OK) return s;
  if (mask && items && (impl == 6 || impl == 0)) {
    const long long entries = attention64_item_entries(g.B, g.H, g.H_kv, g.N);
    a.items = items;
    a.row_counts = items + entries + 2 * g.B * g.H_kv;
    if (impl == 6) return launch_attention64(a, tQa, tK3, tV3, st);  // forced
    // automatic: the density is known on the device only; attention64's pre-pass counts the
    // selected pairs and each kernel's CTAs exit unless attn::m64_wins picks that kernel
    a.sel_pairs = reinterpret_cast<unsigned long long*>(items + entries);
    if ((s = launch_attention64(a, tQa, tK3, tV3, st)) != US_OK) return s;
    a.items = nullptr;
    a.row_counts = nullptr;
  } else if (mask && impl == 6) {
    return launch_attention64(a, tQa, tK3, tV3, st);  // forced, no workspace: the fixed decode order
  }
  return launch_attention(a, tQ, tK3, tV3, st);
}

// ws_ok: the caller's workspace is at least layout(p).total bytes (the attention64 item
// table lives there; without it that kernel walks the fixed decode order).
us_status run_attention(const us_params& p, const void* Q, const void* K, const void* V,
                        const uint32_t* mask, int hpp, void* O, float* lse, cudaStream_t st,
                        uint32_t* err = nullptr, int32_t* first_bad = nullptr, void* ws = nullptr,
                        bool ws_ok = false, bool attn_only = false) {
  Geo g(p);
  us_params q = p;
  int32_t* items = (ws && ws_ok) ? at<int32_t>(ws, layout(p, false, attn_only).items) : nullptr;
  if (p.S == kGpuBlock && p.dtype == US_DTYPE_BF16)
    return run_attention_core(q, Q, K, V, mask, hpp, O, lse, st, err, first_bad, items);
  if (!ws && (p.dtype == US_DTYPE_F32 || (mask && p.S != kGpuBlock))) {
    set_error("attention: f32 inputs / S != 64 need the workspace (us_attention_workspace_bytes)");
    return US_ERR_WORKSPACE;
  }
  Ws w = layout(p, false, attn_only);
  us_status s;
  if (p.S != kGpuBlock) {
    // S = 64 m: the kernels walk 64-row / 64-key sub-blocks of the selected blocks
    q.S = kGpuBlock;
    if (mask) {
      uint32_t* m64 = at<uint32_t>(ws, w.mask64);
      if ((s = launch_mask_expand(mask, (long long)g.B * (g.H / hpp), g.N, g.W, g.S / kGpuBlock, m64, st)) != US_OK)
        return s;
      mask = m64;
    }
  }
  if (p.dtype == US_DTYPE_F32) {
    // the attention kernels compute on bf16 copies of f32 inputs (round to nearest even)
    uint8_t* qb = at<uint8_t>(ws, w.conv);
    uint8_t* kb = qb + size_t(2) * g.B * g.H * g.L * g.D;
    uint8_t* vb = kb + size_t(2) * g.B * g.H_kv * g.L * g.D;
    if ((s = launch_f32_to_bf16(static_cast<const float*>(Q), qb, (long long)g.B * g.H * g.L * g.D, st)) != US_OK)
      return s;
    if ((s = launch_f32_to_bf16(static_cast<const float*>(K), kb, (long long)g.B * g.H_kv * g.L * g.D, st)) != US_OK)
      return s;
    if ((s = launch_f32_to_bf16(static_cast<const float*>(V), vb, (long long)g.B * g.H_kv * g.L * g.D, st)) != US_OK)
      return s;
    q.dtype = US_DTYPE_BF16;
    Q = qb;
    K = kb;
    V = vb;
  }
  return run_attention_core(q, Q, K, V, mask, hpp, O, lse, st, err, first_bad, items);
}


us_status sync_check(const us_params& p, void* ws, cudaStream_t st, const char* who) {
  Ws w = layout(p);
  US_CUDA_TRY(cudaStreamSynchronize(st), "stream synchronize");
  uint32_t hdr[2] = {0, 0};
  US_CUDA_TRY(cudaMemcpy(&hdr[0], at<void>(ws, w.err), 4, cudaMemcpyDeviceToHost), "error word read");
  US_CUDA_TRY(cudaMemcpy(&hdr[1], at<void>(ws, w.first_bad), 4, cudaMemcpyDeviceToHost), "error row read");
  US_CUDA_TRY(cudaMemset(at<void>(ws, w.err), 0, 4), "error word clear");
  const uint32_t err = hdr[0];
  if (err & 1u) {
    set_error("top_p_row: scores must be nonnegative");
    return US_ERR_NONFINITE;
  }
  if (err & 4u) {
    set_error(std::string(who) + ": mask selects a non-causal block");
    return US_ERR_INVALID_MASK;
  }
  if (err & 8u) {
    Geo g(p);
    set_error(std::string(who) + ": query block " + std::to_string(int(hdr[1]) % g.N) +
              " has no selected key block");
    return US_ERR_INVALID_MASK;
  }
  return US_OK;
}

}  // namespace
}  // namespace us

using namespace us;

extern "C" {

const char* us_version(void) { return "unisparse-b200 0.1 (sm_100a)"; }
const char* us_last_error(void) { return g_err.c_str(); }
int32_t us_last_launch_count(void) { return g_launches; }

us_status us_profile_enable(int32_t max_calls) {
  us_profile_disable();
  if (max_calls <= 0) return US_OK;
  g_prof.ev.resize(size_t(max_calls) * 5);
  for (auto& e : g_prof.ev) US_CUDA_TRY(cudaEventCreate(&e), "us_profile_enable");
  g_prof.max_calls = max_calls;
  g_prof.next = 0;
  return US_OK;
}

int32_t us_profile_read(float* ms_out, int32_t max_calls) {
  const int n = std::min(std::min(g_prof.next, g_prof.max_calls), int(max_calls));
  for (int c = 0; c < n; ++c) {
    cudaEventSynchronize(g_prof.ev[size_t(c) * 5 + 4]);
    for (int k = 0; k < 4; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, g_prof.ev[size_t(c) * 5 + k], g_prof.ev[size_t(c) * 5 + k + 1]);
      ms_out[c * 4 + k] = ms;
    }
  }
  return n;
}

void us_profile_disable(void) {
  for (auto& e : g_prof.ev) cudaEventDestroy(e);
  g_prof.ev.clear();
  g_prof.max_calls = 0;
  g_prof.next = 0;
}

int us_validate(const us_params* p, char* msg, size_t cap) {
  if (!p) return 1;
  Checked c = check(*p, true);
  std::vector<std::string> all = c.errors;
  all.insert(all.end(), c.unsupported.begin(), c.unsupported.end());
  if (msg && cap) std::snprintf(msg, cap, "%s", joined(all).c_str());
  return int(all.size());
}

us_status us_set_attention_impl(int32_t impl) {
#ifndef US_CALIBRATION
  if (impl >= 2 && impl <= 5) {
    set_error("us_set_attention_impl: implementations 2-5 are calibration variants, present only in "
              "libunisparse_b200_calib.so");
    return US_ERR_UNSUPPORTED;
  }
#endif
  if (impl < 0 || impl > 6) {
    set_error("us_set_attention_impl: impl must be 0 (automatic), 1 (two query tiles per CTA), 2 (128-key steps), "
              "3 (one tile per CTA), 4 (key-major), 5 (decoupled softmax, P in TMEM) or 6 (one M = 64 chain per "
              "query group)");
    return US_ERR_INVALID_ARGUMENT;
  }
  g_attn_impl.store(impl, std::memory_order_relaxed);
  return US_OK;
}

us_status us_set_attention_pairing(int32_t on) {
  if (on != 0 && on != 1) {
    set_error("us_set_attention_pairing: on must be 0 or 1");
    return US_ERR_INVALID_ARGUMENT;
  }
  g_attn_pairing.store(on, std::memory_order_relaxed);
  return US_OK;
}

us_status us_check_params(const us_params* p, const char* who, int32_t need_compression) {
  return gate(p, who ? who : "us_check_params", need_compression != 0);
}

size_t us_workspace_bytes(const us_params* p) {
  if (!p || !check(*p, false).errors.empty()) return 0;
  if (needs_pad(*p) && p->d_k <= 128) return padded_ws_bytes(*p);
  return layout(*p).total;
}

size_t us_attention_workspace_bytes(const us_params* p) {
  if (!p || !check(*p, false).errors.empty()) return 0;
  if (needs_pad(*p) && p->d_k <= 128) return padded_ws_bytes(*p, true);
  return layout(*p, false, true).total;
}

us_status us_compress(const us_params* p, const void* Q, const void* K, float* Qc, float* Kc,
                      void* workspace, size_t workspace_bytes, void* stream) {
  (void)workspace;
  (void)workspace_bytes;
  us_status s = gate(p, "compress", true);
  if (s != US_OK) return s;
  Geo g(*p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "compress", ps)) != US_OK) return s;
    if ((s = pad_inputs(*p, ps, Q, K, nullptr, st)) != US_OK) return s;
    float* qc = reinterpret_cast<float*>(ps.base + ps.w.qc);
    float* kc = reinterpret_cast<float*>(ps.base + ps.w.kc);
    if ((s = us_compress(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, qc, kc, workspace, ps.inner_bytes, stream)) !=
        US_OK)
      return s;
    if ((s = unpad_rows(qc, Qc, size_t(g.B) * g.Hc * g.Lq, g.D, ps.pp.d_k, 4, st)) != US_OK) return s;
    if ((s = unpad_rows(kc, Kc, size_t(g.B) * g.Hc * g.Lk, g.D, ps.pp.d_k, 4, st)) != US_OK) return s;
    if (p->flags & US_FLAG_SYNC_CHECK) US_CUDA_TRY(cudaStreamSynchronize(st), "compress");
    return US_OK;
  }
  // reference layout: H/c_h planes for both Q and K (K expanded to H heads first)
  CompressArgs cq{static_cast<const uint16_t*>(Q), g.B, g.H, g.L, g.D, p->c_q, g.Hc, p->c_h, 1, Qc, nullptr,
                  p->strategy, 0, p->seed, p->head0, nullptr, nullptr, nullptr, p->dtype == US_DTYPE_F32};
  if ((s = launch_compress(cq, st)) != US_OK) return s;
  CompressArgs ck{static_cast<const uint16_t*>(K), g.B, g.H_kv, g.L, g.D, p->c_k, g.Hc, p->c_h, g.G, Kc, nullptr,
                  p->strategy, 1, p->seed, p->head0, nullptr, nullptr, nullptr, p->dtype == US_DTYPE_F32};
  if ((s = launch_compress(ck, st)) != US_OK) return s;
  if (p->flags & US_FLAG_SYNC_CHECK) US_CUDA_TRY(cudaStreamSynchronize(st), "compress");
  return US_OK;
}

us_status us_select(const us_params* p, const void* Q, const void* K, const us_selection* out,
                    void* workspace, size_t workspace_bytes, void* stream) {
  us_status s = gate(p, "select_blocks", true);
  if (s != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "select_blocks", ps)) != US_OK) return s;
    if ((s = pad_inputs(*p, ps, Q, K, nullptr, st)) != US_OK) return s;
    ScaleDk scale(p->d_k);
    return us_select(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, out, workspace, ps.inner_bytes, stream);
  }
  if ((s = need_ws(*p, workspace, workspace_bytes, "select_blocks")) != US_OK) return s;
  Geo g(*p);
  Ws w = layout(*p);
  ProxyArgs pa{};
  if ((s = run_proxy(*p, Q, K, workspace, st, &pa)) != US_OK) return s;
  uint32_t* mask = (out && out->mask_bits) ? out->mask_bits : at<uint32_t>(workspace, w.mask);
  if ((s = run_select_fused(*p, pa, mask, out, workspace, st)) != US_OK) return s;
  if (p->flags & US_FLAG_SYNC_CHECK) return sync_check(*p, workspace, st, "select_blocks");
  return US_OK;
}

size_t us_proxy_workspace_bytes(const us_params* p, int32_t proxy, int32_t stride) {
  if (!p || !check(*p, false).errors.empty()) return 0;
  if (proxy == US_PROXY_ANTIDIAGONAL && stride > 0) return layout(antidiag_params(*p, stride), true).total;
  if (proxy == US_PROXY_LAST_BLOCK) return layout(antidiag_params(*p, p->S), true).total;
  return us_workspace_bytes(p);
}

us_status us_select_proxy(const us_params* p, int32_t proxy, int32_t stride, const void* Q, const void* K,
                          const us_selection* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (proxy == US_PROXY_UNISPARSE) return us_select(p, Q, K, out, workspace, workspace_bytes, stream);
  if (p && needs_pad(*p) && p->d_k <= 128) {
    set_error("select_blocks: d_k=" + std::to_string(p->d_k) +
              " is supported by the UniSparse proxy only on the GPU path (competitor proxies: 64 or 128)");
    return US_ERR_UNSUPPORTED;
  }
  us_status s = gate(p, "select_blocks", false);
  if (s != US_OK) return s;
  if (proxy == US_PROXY_LAST_BLOCK) {
    // last_block_probe_scores (baselines.cpp:54-87), planes = H. Workspace: the
    // layout of one composite row per block (c = S); the chunk statistics, row LSE
    // and column masses live in its (large) slot-partial region.
    const us_params q = antidiag_params(*p, p->S);
    if ((s = need_ws(q, workspace, workspace_bytes, "select_blocks", true)) != US_OK) return s;
    Geo g(q);
    Ws w = layout(q, true);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    US_CUDA_TRY(cudaMemsetAsync(workspace, 0, w.header_bytes, st), "workspace clear");
    LastBlockArgs la{};
    la.B = g.B;
    la.H = g.H;
    la.H_kv = g.H_kv;
    la.L = g.L;
    la.N = g.N;
    la.D = g.D;
    la.Q = static_cast<const uint16_t*>(Q);
    la.K = static_cast<const uint16_t*>(K);
    la.scale_log2 = float(1.4426950408889634 / std::sqrt(double(g.Ds)));
    const size_t stat = size_t(g.B) * g.H * (g.L / 256) * 64;
    la.cmax = at<float>(workspace, w.part);
    la.csum = la.cmax + stat;
    la.lse2 = la.csum + stat;
    la.colmass = la.lse2 + size_t(g.B) * g.H * 64;
    la.scores = at<float>(workspace, w.scores);
    if ((s = launch_last_block_probe(la, st)) != US_OK) return s;
    if (out && out->scores)
      US_CUDA_TRY(cudaMemcpyAsync(out->scores, la.scores, size_t(4) * g.B * g.H * g.N * g.N,
                                  cudaMemcpyDeviceToDevice, st),
                  "scores copy");
    uint32_t* mask = (out && out->mask_bits) ? out->mask_bits : at<uint32_t>(workspace, w.mask);
    if ((s = run_select_rows(q, la.scores, g.H, mask, out, workspace, st)) != US_OK) return s;
    if (p->flags & US_FLAG_SYNC_CHECK) return sync_check(q, workspace, st, "select_blocks");
    return US_OK;
  }
  if (proxy != US_PROXY_ANTIDIAGONAL) {
    set_error("select_blocks: unknown proxy");
    return US_ERR_INVALID_ARGUMENT;
  }
  if (stride <= 0 || p->S % stride != 0) {
    set_error("antidiagonal_block_scores: stride must divide S");
    return US_ERR_INVALID_ARGUMENT;
  }
  if (!is_pow2(p->S / stride) || p->S / stride > 64) {
    set_error("select_blocks: S/stride must be a power of two on the GPU path");
    return US_ERR_UNSUPPORTED;
  }
  const us_params q = antidiag_params(*p, stride);
  if ((s = need_ws(q, workspace, workspace_bytes, "select_blocks", true)) != US_OK) return s;
  Geo g(q);
  Ws w = layout(q, true);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  US_CUDA_TRY(cudaMemsetAsync(workspace, 0, w.header_bytes, st), "workspace clear");
  if ((s = run_antidiagonal(*p, stride, Q, K, workspace, st)) != US_OK) return s;
  if (out && out->scores)
    US_CUDA_TRY(cudaMemcpyAsync(out->scores, at<float>(workspace, w.scores), size_t(4) * g.B * g.H * g.N * g.N,
                                cudaMemcpyDeviceToDevice, st),
                "scores copy");
  uint32_t* mask = (out && out->mask_bits) ? out->mask_bits : at<uint32_t>(workspace, w.mask);
  if ((s = run_select_rows(q, at<float>(workspace, w.scores), g.H, mask, out, workspace, st)) != US_OK) return s;
  if (p->flags & US_FLAG_SYNC_CHECK) return sync_check(q, workspace, st, "select_blocks");
  return US_OK;
}

// ---------------------------------------------------------------- quality metrics (§8f-4)
size_t us_mass_workspace_bytes(const us_params* p) {
  if (!p || !check(*p, false).errors.empty()) return 0;
  if (needs_pad(*p) && p->d_k <= 128)
    return al(layout(antidiag_params(padded_params(*p), 1), true).total) + pad_layout(*p).total;
  return layout(antidiag_params(*p, 1), true).total;
}

us_status us_exact_block_mass(const us_params* p, const void* Q, const void* K, float* mass, void* workspace,
                              size_t workspace_bytes, void* stream) {
  // exact_block_mass (attention.cpp:56-86) = the strided scorer at stride 1: every
  // query row against its causal keys (live = r + 1), bf16 products accumulated in
  // fp32, row softmax, block sums — the proxy kernel's raw-input mode.
  us_status s = gate(p, "exact_block_mass", false);
  if (s != US_OK) return s;
  if (!mass) {
    set_error("exact_block_mass: null output");
    return US_ERR_INVALID_ARGUMENT;
  }
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "exact_block_mass", ps,
                       layout(antidiag_params(padded_params(*p), 1), true).total)) != US_OK)
      return s;
    if ((s = pad_inputs(*p, ps, Q, K, nullptr, static_cast<cudaStream_t>(stream))) != US_OK) return s;
    ScaleDk scale(p->d_k);
    return us_exact_block_mass(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, mass, workspace, ps.inner_bytes, stream);
  }
  const us_params q = antidiag_params(*p, 1);
  if ((s = need_ws(q, workspace, workspace_bytes, "exact_block_mass", true)) != US_OK) return s;
  Geo g(q);
  Ws w = layout(q, true);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  US_CUDA_TRY(cudaMemsetAsync(workspace, 0, w.header_bytes, st), "workspace clear");
  if ((s = run_antidiagonal(*p, 1, Q, K, workspace, st)) != US_OK) return s;
  US_CUDA_TRY(cudaMemcpyAsync(mass, at<float>(workspace, w.scores), size_t(4) * g.B * g.H * g.N * g.N,
                              cudaMemcpyDeviceToDevice, st),
              "mass copy");
  return launch_fill_upper(mass, (long long)g.B * g.H, g.N, st);
}

size_t us_metrics_workspace_bytes(const us_params* p) {
  if (!p || !check(*p, false).errors.empty()) return 0;
  const size_t rows_l = size_t(p->B) * p->H * p->L, rows_n = size_t(p->B) * p->H * (p->L / p->S);
  return 256 + std::max(24 * rows_l, 9 * rows_n + 256);
}

namespace {
us_status metrics_ws(const us_params* p, void* ws, size_t bytes, const char* who) {
  const size_t need = us_metrics_workspace_bytes(p);
  if (!ws || bytes < need) {
    set_error(std::string(who) + ": workspace of " + std::to_string(need) + " bytes required");
    return US_ERR_WORKSPACE;
  }
  return US_OK;
}
}  // namespace

us_status us_output_fidelity(const us_params* p, const void* O_test, const void* O_ref, double* out3,
                             void* workspace, size_t workspace_bytes, void* stream) {
  us_status s = gate(p, "output_fidelity", false);
  if (s != US_OK) return s;
  if (!O_test || !O_ref || !out3) {
    set_error("output_fidelity: null argument");
    return US_ERR_INVALID_ARGUMENT;
  }
  if ((s = metrics_ws(p, workspace, workspace_bytes, "output_fidelity")) != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* res = at<double>(workspace, 0);
  const long long rows = (long long)p->B * p->H * p->L;
  if ((s = launch_output_fidelity(rows, p->d_k, static_cast<const uint16_t*>(O_test),
                                  static_cast<const uint16_t*>(O_ref), at<double>(workspace, 256), res, st)) != US_OK)
    return s;
  US_CUDA_TRY(cudaMemcpyAsync(out3, res, 3 * sizeof(double), cudaMemcpyDeviceToHost, st), "fidelity readback");
  US_CUDA_TRY(cudaStreamSynchronize(st), "output_fidelity");
  return US_OK;
}

us_status us_block_recall(const us_params* p, const uint32_t* mask_bits, int32_t heads_per_plane, const float* ref,
                          int32_t k, double* out, void* workspace, size_t workspace_bytes, void* stream) {
  us_status s = gate(p, "block_recall", false);
  if (s != US_OK) return s;
  const int N = p->L / p->S;
  if (k < 1 || k > N) {
    set_error("block_recall: k out of range");
    return US_ERR_INVALID_ARGUMENT;
  }
  if (heads_per_plane <= 0 || p->H % heads_per_plane != 0 || !mask_bits || !ref || !out) {
    set_error("block_recall: reference must hold one plane per mask head");
    return US_ERR_INVALID_ARGUMENT;
  }
  if ((s = metrics_ws(p, workspace, workspace_bytes, "block_recall")) != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* res = at<double>(workspace, 0);
  if ((s = launch_block_recall(p->B, p->H, N, (N + 31) / 32, p->H / heads_per_plane, heads_per_plane, k, mask_bits,
                               ref, at<double>(workspace, 256), res, st)) != US_OK)
    return s;
  US_CUDA_TRY(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, st), "recall readback");
  US_CUDA_TRY(cudaStreamSynchronize(st), "block_recall");
  return US_OK;
}

us_status us_planted_recall(const us_params* p, const uint32_t* mask_bits, int32_t heads_per_plane,
                            const int32_t* planted, int32_t m, double* out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  us_status s = gate(p, "planted_recall", false);
  if (s != US_OK) return s;
  if (!planted || m <= 0 || !mask_bits || !out || heads_per_plane <= 0 || p->H % heads_per_plane != 0) {
    set_error("planted_recall: planted must hold one list set per head");
    return US_ERR_INVALID_ARGUMENT;
  }
  if ((s = metrics_ws(p, workspace, workspace_bytes, "planted_recall")) != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int N = p->L / p->S;
  const long long rows = (long long)p->B * p->H * N;
  double* res = at<double>(workspace, 0);
  long long* ndef = at<long long>(workspace, 64);
  double* row_val = at<double>(workspace, 256);
  uint8_t* def = reinterpret_cast<uint8_t*>(row_val + rows);
  if ((s = launch_planted_recall(p->B, p->H, N, (N + 31) / 32, p->H / heads_per_plane, heads_per_plane, m, mask_bits,
                                 planted, row_val, def, res, ndef, st)) != US_OK)
    return s;
  long long host_def = 0;
  US_CUDA_TRY(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, st), "planted readback");
  US_CUDA_TRY(cudaMemcpyAsync(&host_def, ndef, sizeof(long long), cudaMemcpyDeviceToHost, st), "planted readback");
  US_CUDA_TRY(cudaStreamSynchronize(st), "planted_recall");
  if (host_def == 0) {
    set_error("planted_recall: no planted rows");
    return US_ERR_INVALID_ARGUMENT;
  }
  return US_OK;
}

us_status us_mean_row_spearman(const us_params* p, const float* proxy, const float* ref, double* mean,
                               int64_t* defined, int64_t* undefined, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (p && (p->c_h <= 0 || p->H <= 0 || p->H % p->c_h != 0)) {
    set_error("mean_row_spearman: head counts disagree");
    return US_ERR_INVALID_ARGUMENT;
  }
  us_status s = gate(p, "mean_row_spearman", false);
  if (s != US_OK) return s;
  if (!proxy || !ref || !mean) {
    set_error("mean_row_spearman: null argument");
    return US_ERR_INVALID_ARGUMENT;
  }
  if ((s = metrics_ws(p, workspace, workspace_bytes, "mean_row_spearman")) != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int N = p->L / p->S;
  const long long rows = (long long)p->B * p->H * N;
  double* res = at<double>(workspace, 0);
  long long* ndef = at<long long>(workspace, 64);
  double* row_val = at<double>(workspace, 256);
  uint8_t* def = reinterpret_cast<uint8_t*>(row_val + rows);
  if ((s = launch_row_spearman(p->B, p->H, N, p->c_h, proxy, ref, row_val, def, res, ndef, st)) != US_OK) return s;
  long long host_def = 0;
  US_CUDA_TRY(cudaMemcpyAsync(mean, res, sizeof(double), cudaMemcpyDeviceToHost, st), "spearman readback");
  US_CUDA_TRY(cudaMemcpyAsync(&host_def, ndef, sizeof(long long), cudaMemcpyDeviceToHost, st), "spearman readback");
  US_CUDA_TRY(cudaStreamSynchronize(st), "mean_row_spearman");
  // rows i = 1 .. N-1 of every (b, h) are scored; the rest of the count is undefined
  const long long scored = (long long)p->B * p->H * (N - 1);
  if (defined) *defined = host_def;
  if (undefined) *undefined = scored - host_def;
  return US_OK;
}

us_status us_build_block_mask(const us_params* p, const float* scores, const us_selection* out,
                              void* workspace, size_t workspace_bytes, void* stream) {
  us_status s = gate(p, "build_block_mask", false);
  if (s != US_OK) return s;
  if ((s = need_ws(*p, workspace, workspace_bytes, "build_block_mask")) != US_OK) return s;
  if (!out || !out->mask_bits) {
    set_error("build_block_mask: out->mask_bits is required");
    return US_ERR_INVALID_ARGUMENT;
  }
  Geo g(*p);
  Ws w = layout(*p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  US_CUDA_TRY(cudaMemsetAsync(workspace, 0, w.header_bytes, st), "workspace clear");
  if ((s = run_select_rows(*p, scores, g.Hc, out->mask_bits, out, workspace, st)) != US_OK) return s;
  if (p->flags & US_FLAG_SYNC_CHECK) return sync_check(*p, workspace, st, "build_block_mask");
  return US_OK;
}

us_status us_sparse_attention(const us_params* p, const void* Q, const void* K, const void* V,
                              const uint32_t* mask_bits, int32_t heads_per_plane, void* O,
                              float* lse, void* workspace, size_t workspace_bytes, void* stream) {
  us_status s = gate(p, "block_sparse_attention", false);
  if (s != US_OK) return s;
  if (heads_per_plane <= 0 || p->H % heads_per_plane != 0) {
    set_error("block_sparse_attention: heads_per_plane must divide H");
    return US_ERR_INVALID_ARGUMENT;
  }
  if (!mask_bits) {
    set_error("block_sparse_attention: mask_bits is required");
    return US_ERR_INVALID_ARGUMENT;
  }
  Geo g(*p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "block_sparse_attention", ps,
                       layout(padded_params(*p), false, true).total)) != US_OK)
      return s;
    if ((s = pad_inputs(*p, ps, Q, K, V, st)) != US_OK) return s;
    {
      ScaleDk scale(p->d_k);
      if ((s = us_sparse_attention(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, ps.base + ps.w.v, mask_bits,
                                   heads_per_plane, ps.base + ps.w.o, lse, workspace, ps.inner_bytes, stream)) != US_OK)
        return s;
    }
    if ((s = unpad_rows(ps.base + ps.w.o, O, size_t(g.B) * g.H * g.L, g.D, ps.pp.d_k, 2, st)) != US_OK) return s;
    if (p->flags & US_FLAG_SYNC_CHECK) US_CUDA_TRY(cudaStreamSynchronize(st), "block_sparse_attention");
    return US_OK;
  }
  if (p->flags & US_FLAG_SYNC_CHECK) {
    if ((s = need_ws(*p, workspace, workspace_bytes, "block_sparse_attention", false, true)) != US_OK) return s;
    Ws w = layout(*p, false, true);
    US_CUDA_TRY(cudaMemsetAsync(workspace, 0, 4, st), "workspace clear");
    US_CUDA_TRY(cudaMemsetAsync(at<uint8_t>(workspace, w.first_bad), 0x7F, 4, st), "workspace clear");
    if ((s = launch_mask_check(mask_bits, g.B * (g.H / heads_per_plane) * g.N, g.N, g.W,
                               at<uint32_t>(workspace, w.err), at<int32_t>(workspace, w.first_bad), st)) != US_OK)
      return s;
    if ((s = sync_check(*p, workspace, st, "block_sparse_attention")) != US_OK) return s;
  }
  if ((p->dtype == US_DTYPE_F32 || p->S != kGpuBlock) &&
      (s = need_ws(*p, workspace, workspace_bytes, "block_sparse_attention", false, true)) != US_OK)
    return s;
  uint32_t* err = nullptr;
  int32_t* first_bad = nullptr;
  if (workspace && workspace_bytes >= layout(*p, false, true).total) {
    // asynchronous data-error report (us_check_device_errors): the kernel ORs 4 (a
    // non-causal bit) or 8 (an empty row) into the sticky error word and records the
    // first offending row, as the reference throws (attention.cpp:106-108, 127-129)
    Ws w = layout(*p, false, true);
    err = at<uint32_t>(workspace, w.err);
    first_bad = at<int32_t>(workspace, w.first_bad);
    US_CUDA_TRY(cudaMemsetAsync(first_bad, 0x7F, 4, st), "workspace clear");
  }
  if ((s = run_attention(*p, Q, K, V, mask_bits, heads_per_plane, O, lse, st, err, first_bad, workspace,
                         workspace && workspace_bytes >= layout(*p, false, true).total, true)) != US_OK)
    return s;
  if (p->flags & US_FLAG_SYNC_CHECK) US_CUDA_TRY(cudaStreamSynchronize(st), "block_sparse_attention");
  return US_OK;
}

us_status us_unisparse_attention(const us_params* p, const void* Q, const void* K, const void* V,
                                 void* O, float* lse, const us_selection* sel, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  // unisparse_attn validates through select_blocks (pipeline.cpp:19-24 -> :7-8)
  us_status s = gate(p, "select_blocks", true);
  if (s != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "unisparse_attn", ps)) != US_OK) return s;
    if ((s = pad_inputs(*p, ps, Q, K, V, st)) != US_OK) return s;
    {
      ScaleDk scale(p->d_k);
      if ((s = us_unisparse_attention(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, ps.base + ps.w.v, ps.base + ps.w.o,
                                      lse, sel, workspace, ps.inner_bytes, stream)) != US_OK)
        return s;
    }
    Geo g(*p);
    return unpad_rows(ps.base + ps.w.o, O, size_t(g.B) * g.H * g.L, g.D, ps.pp.d_k, 2, st);
  }
  if ((s = need_ws(*p, workspace, workspace_bytes, "unisparse_attn")) != US_OK) return s;
  Geo g(*p);
  Ws w = layout(*p);
  const int call = g_prof.on() ? g_prof.next++ : -1;
  g_prof.mark(call, 0, st);
  ProxyArgs pa{};
  if ((s = run_proxy(*p, Q, K, workspace, st, &pa, call)) != US_OK) return s;
  g_prof.mark(call, 2, st);
  uint32_t* mask = (sel && sel->mask_bits) ? sel->mask_bits : at<uint32_t>(workspace, w.mask);
  if ((s = run_select_fused(*p, pa, mask, sel, workspace, st)) != US_OK) return s;
  g_prof.mark(call, 3, st);
  if ((s = run_attention(*p, Q, K, V, mask, p->c_h, O, lse, st, nullptr, nullptr, workspace, true)) != US_OK)
    return s;
  g_prof.mark(call, 4, st);
  if (p->flags & US_FLAG_SYNC_CHECK) return sync_check(*p, workspace, st, "unisparse_attn");
  return US_OK;
}

us_status us_dense_attention(const us_params* p, const void* Q, const void* K, const void* V,
                             void* O, float* lse, void* workspace, size_t workspace_bytes,
                             void* stream) {
  us_status s = gate(p, "dense_attention", false);
  if (s != US_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (needs_pad(*p)) {
    PadStage ps;
    if ((s = pad_begin(*p, workspace, workspace_bytes, "dense_attention", ps,
                       layout(padded_params(*p), false, true).total)) != US_OK)
      return s;
    if ((s = pad_inputs(*p, ps, Q, K, V, st)) != US_OK) return s;
    {
      ScaleDk scale(p->d_k);
      if ((s = us_dense_attention(&ps.pp, ps.base + ps.w.q, ps.base + ps.w.k, ps.base + ps.w.v, ps.base + ps.w.o, lse,
                                  workspace, ps.inner_bytes, stream)) != US_OK)
        return s;
    }
    Geo g(*p);
    return unpad_rows(ps.base + ps.w.o, O, size_t(g.B) * g.H * g.L, g.D, ps.pp.d_k, 2, st);
  }
  if (p->dtype == US_DTYPE_F32 && (s = need_ws(*p, workspace, workspace_bytes, "dense_attention", false, true)) != US_OK) return s;
  if ((s = run_attention(*p, Q, K, V, nullptr, 1, O, lse, st, nullptr, nullptr, workspace, false, true)) != US_OK)
    return s;
  if (p->flags & US_FLAG_SYNC_CHECK) US_CUDA_TRY(cudaStreamSynchronize(st), "dense_attention");
  return US_OK;
}

us_status us_check_device_errors(const us_params* p, void* workspace, void* stream) {
  if (!p || !workspace) {
    set_error("us_check_device_errors: null argument");
    return US_ERR_INVALID_ARGUMENT;
  }
  return sync_check(*p, workspace, static_cast<cudaStream_t>(stream), "unisparse_attn");
}

us_status us_selection_flops(const us_params* p, int32_t proxy, int32_t stride, uint64_t* f) {
  // metrics.cpp:44-81 (exact u64)
  if (!p || !f) return US_ERR_INVALID_ARGUMENT;
  const uint64_t L = uint64_t(p->L), H = uint64_t(p->H), d = uint64_t(p->d_k), S = uint64_t(p->S);
  if (p->L <= 0 || p->H <= 0 || p->d_k <= 0 || p->S <= 0 || L % S != 0) {
    set_error("selection_flops: bad dimensions");
    return US_ERR_INVALID_ARGUMENT;
  }
  const uint64_t N = L / S;
  uint64_t lg = 0;
  while ((uint64_t(1) << lg) < N) ++lg;
  for (int t = 0; t < 6; ++t) f[t] = 0;
  f[5] = 4 * L * L * H * d;
  if (proxy == US_PROXY_UNISPARSE) {
    if (p->c_q <= 0 || p->c_k <= 0 || p->c_h <= 0 || S % uint64_t(p->c_q) || S % uint64_t(p->c_k) ||
        H % uint64_t(p->c_h)) {
      set_error("selection_flops: bad compression factors");
      return US_ERR_INVALID_ARGUMENT;
    }
    const uint64_t cq = p->c_q, ck = p->c_k, ch = p->c_h;
    f[0] = 2 * L * H * d + (ch > 1 ? 2 * (L / cq + L / ck) * H * d : 0);
    f[1] = 2 * (L / cq) * (L / ck) * (H / ch) * d;
    f[2] = 4 * (L / cq) * (L / ck) * (H / ch);
    f[3] = (H / ch) * N * N * lg;
  } else if (proxy == US_PROXY_ANTIDIAGONAL) {
    if (stride <= 0 || S % uint64_t(stride)) {
      set_error("selection_flops: stride must divide S");
      return US_ERR_INVALID_ARGUMENT;
    }
    f[1] = 2 * L * (L / stride) * H * d;
    f[2] = 2 * L * (L / stride) * H;
    f[3] = H * N * N * lg;
  } else {
    f[1] = 2 * S * L * H * d;
    f[2] = 2 * S * L * H;
    f[3] = H * N * N * lg;
  }
  return US_OK;
}

}  // extern "C"
