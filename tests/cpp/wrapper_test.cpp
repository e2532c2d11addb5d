// wrapper_test.cpp — the C++ mirror (include/unisparse_b200.hpp) exercised the
// way the reference's own doctest suites exercise unisparse:: (test
// infrastructure; built by __graft_entry__.build() into
// paper_2512_14082_b200/_build/wrapper_test).
//
//   wrapper_test cpu   — no device work: validation text and exception types
//                         (types.cpp:97-123, pipeline.cpp:7-8), pinned FLOP
//                         integers (test_metrics.cpp:224-270)
//   wrapper_test gpu   — unisparse_attn / select_blocks / block_sparse_attention /
//                         dense_attention on a small planted-like input: P = 1 is
//                         dense (test_pipeline.cpp:9-21), the report is
//                         consistent with the mask, sparse attention on the
//                         selected mask reproduces unisparse_attn bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "unisparse_b200.hpp"

namespace u = unisparse_b200;

static int g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static std::string expect_throw(F&& f) {
  try {
    f();
  } catch (const E& e) {
    return e.what();
  } catch (const std::exception& e) {
    return std::string("WRONG TYPE: ") + e.what();
  }
  return "NO THROW";
}

static void cpu_tests() {
  u::AttentionInputs in;
  in.H = 4;
  in.L = 1000;
  in.d_k = 64;
  in.S = 64;
  u::CompressionConfig cfg;
  std::string m = expect_throw<std::invalid_argument>([&] { u::unisparse_attn(in, cfg); });
  CHECK(m == "select_blocks: L=1000 not divisible by S=64");
  m = expect_throw<std::invalid_argument>([&] { u::select_blocks(in, cfg); });
  CHECK(m == "select_blocks: L=1000 not divisible by S=64");
  m = expect_throw<std::invalid_argument>([&] { u::compress(in, cfg); });
  CHECK(m == "compress: L=1000 not divisible by S=64");
  // collect-all, reference order (types.cpp:97-123)
  in.L = 1024;
  in.H = 6;
  cfg.c_q = 3;
  cfg.c_h = 4;
  m = expect_throw<std::invalid_argument>([&] { u::select_blocks(in, cfg); });
  CHECK(m == "select_blocks: S=64 not divisible by c_q=3; H=6 not divisible by c_h=4");
  cfg = u::CompressionConfig();
  cfg.P = 0.0;
  in.H = 4;
  m = expect_throw<std::invalid_argument>([&] { u::select_blocks(in, cfg); });
  CHECK(m == "select_blocks: P must lie in (0, 1]");
  in.d_k = 0;
  m = expect_throw<std::invalid_argument>([&] { u::dense_attention(in); });
  CHECK(m == "dense_attention: d_k must be positive");
  // valid for the reference, outside the GPU path: domain_error, not invalid_argument
  // (d_k <= 128 runs zero-padded; above 128 is outside the GPU path)
  in.d_k = 160;
  cfg = u::CompressionConfig();
  m = expect_throw<std::domain_error>([&] { u::select_blocks(in, cfg); });
  CHECK(m.find("unsupported on the GPU path") != std::string::npos);

  // pinned FLOP integers (test_metrics.cpp:224-247)
  u::CompressionConfig c8;
  u::FlopBreakdown f = u::selection_flops(4096, 4, 64, 128, c8);
  CHECK(f.compression == 2097152ull);
  CHECK(f.compressed_qk == 134217728ull);
  CHECK(f.softmax_aggregation == 4194304ull);
  CHECK(f.top_p == 20480ull);
  CHECK(f.dense_attention == 17179869184ull);
  c8.c_h = 2;
  f = u::selection_flops(4096, 4, 64, 128, c8);
  CHECK(f.compressed_qk == 67108864ull);
  CHECK(f.softmax_aggregation == 2097152ull);
  CHECK(f.top_p == 10240ull);
  CHECK(f.compression == 2097152ull + 524288ull);
  std::printf("cpu: %s\n", g_fail ? "FAILED" : "ok");
}

static uint16_t to_bf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
static float from_bf16(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

static void gpu_tests() {
  const int B = 1, H = 8, H_kv = 2, L = 2048, d = 128, S = 64, N = L / S;
  std::mt19937_64 rng(2512);
  std::normal_distribution<float> nd(0.f, 0.1f);
  std::vector<uint16_t> q(size_t(B) * H * L * d), k(size_t(B) * H_kv * L * d), v(k.size());
  // planted-style structure: query block i of head h and two earlier key blocks share a direction
  std::vector<float> qf(q.size()), kf(k.size());
  for (auto& x : qf) x = nd(rng);
  for (auto& x : kf) x = nd(rng);
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      std::vector<float> dir(d);
      float nrm = 0.f;
      for (auto& x : dir) {
        x = nd(rng);
        nrm += x * x;
      }
      nrm = std::sqrt(nrm);
      const int j = int(rng() % uint64_t(i + 1));
      for (int t = 0; t < S; ++t)
        for (int c = 0; c < d; ++c) {
          qf[((size_t(h) * L) + i * S + t) * d + c] += 8.f * dir[c] / nrm;
          kf[((size_t(h / (H / H_kv)) * L) + j * S + t) * d + c] += 8.f * dir[c] / nrm / 4.f;
        }
    }
  for (size_t t = 0; t < q.size(); ++t) q[t] = to_bf16(qf[t]);
  for (size_t t = 0; t < k.size(); ++t) k[t] = to_bf16(kf[t]);
  for (auto& x : v) x = to_bf16(nd(rng));
  u::DeviceBuffer<uint16_t> dq(q.size()), dk(k.size()), dv(v.size());
  cudaMemcpy(dq.data(), q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dk.data(), k.data(), k.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dv.data(), v.data(), v.size() * 2, cudaMemcpyHostToDevice);
  u::AttentionInputs in;
  in.B = B;
  in.H = H;
  in.H_kv = H_kv;
  in.L = L;
  in.d_k = d;
  in.S = S;
  in.Q = dq.data();
  in.K = dk.data();
  in.V = dv.data();

  // P = 1 selects every causal block: rho = 0, output == dense (test_pipeline.cpp:9-21)
  u::CompressionConfig full;
  full.P = 1.0;
  u::UniSparseResult r1 = u::unisparse_attn(in, full);
  CHECK(std::fabs(r1.report.rho_mean) < 1e-15);
  CHECK(r1.report.mask.selected_total() == int64_t(H) * N * (N + 1) / 2);
  u::AttentionOutput dense = u::dense_attention(in);
  {
    // same function through two kernels (key-major sparse, query-major dense): bf16 agreement
    const auto x1 = r1.out.O.to_host(), xd = dense.O.to_host();
    double worst = 0;
    for (size_t t = 0; t < x1.size(); ++t)
      worst = std::max(worst, double(std::fabs(from_bf16(x1[t]) - from_bf16(xd[t]))));
    CHECK(worst <= 2e-2);
  }

  // P = 0.95: report consistent with the mask; block_sparse_attention on that
  // mask reproduces unisparse_attn bit for bit; selection is monotone in P
  u::CompressionConfig cfg;
  u::UniSparseResult r = u::unisparse_attn(in, cfg);
  int64_t sel = 0;
  for (auto s : r.report.selected) sel += s;
  CHECK(sel == r.report.mask.selected_total());
  CHECK(r.report.rho_mean > 0.0 && r.report.rho_mean < 1.0);
  CHECK(r.report.flops.sparse_attention == uint64_t(sel) * 4ull * S * S * d);
  u::AttentionOutput o2 = u::block_sparse_attention(in, r.report.mask);
  CHECK(o2.O.to_host() == r.out.O.to_host());
  u::CompressionConfig c9;
  c9.P = 0.9;
  u::SparsityReport r9 = u::select_blocks(in, c9);
  CHECK(r9.mask.selected_total() <= sel);
  // sparse output stays close to dense on planted data (cosine criterion 5 analogue)
  const auto a = r.out.O.to_host(), bq = dense.O.to_host();
  double dot = 0, na = 0, nb = 0;
  for (size_t t = 0; t < a.size(); ++t) {
    const double x = from_bf16(a[t]), y = from_bf16(bq[t]);
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  const double cosv = dot / std::sqrt(na * nb);
  CHECK(cosv > 0.9);
  // competitor proxies through the same selection machinery (test_baselines.cpp:157-183)
  for (u::ProxyTag tag : {u::ProxyTag::Antidiagonal, u::ProxyTag::LastBlockProbe}) {
    u::SparsityReport rp = u::select_blocks(tag, in, cfg, 8);
    CHECK(rp.mask.H == H && rp.mask.c_h == 1);
    CHECK(rp.mask.selected_total() >= int64_t(H) * N);  // every causal row keeps >= 1 block
  }
  std::printf("gpu: rho=%.4f selected=%lld cos(sparse,dense)=%.5f %s\n", r.report.rho_mean, (long long)sel,
              cosv, g_fail ? "FAILED" : "ok");
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu" || mode == "all") cpu_tests();
  if (mode == "gpu" || mode == "all") gpu_tests();
  return g_fail ? 1 : 0;
}
