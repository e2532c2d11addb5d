// oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.h for scope and citations).
//
// Plain-loop fp64 restatement of the UniSparse reference hot path. Compiled
// with -ffp-contract=off and without -ffast-math so every fp64 operation is a
// separately rounded IEEE op in a fixed, documented order:
//   * dot products: 8 interleaved fp64 partial sums over the d index
//     (lane = c % 8), combined pairwise ((0+1)+(2+3))+((4+5)+(6+7)).
//     The reference's Eigen GEMM order is unknown; this only moves results in
//     the last bits.
//   * every other reduction (window sums, softmax denominators, region sums,
//     Top-P cumulative sums) is sequential in index order, as in the
//     reference's own naive oracles (tests/oracles.hpp).
#include "oracle.h"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;
int fail(const std::string& msg) {
  g_err = msg;
  return 1;
}

constexpr double kMaskedScore = -double(FLT_MAX);  // types.hpp:32
constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;  // rng.hpp:11

inline uint64_t mix64(uint64_t z) {  // rng.hpp:13-17
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t chain(uint64_t s, uint64_t a) { return mix64(s + kGamma + a); }  // rng.hpp:20-22
inline uint64_t chain(uint64_t s, uint64_t a, uint64_t b) { return chain(chain(s, a), b); }
inline uint64_t chain(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return chain(chain(s, a, b), c);
}

struct Rng {  // rng.hpp:33-67 (CounterRng)
  uint64_t state;
  double spare = 0.0;
  bool have_spare = false;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next_u64() {
    state += kGamma;
    return mix64(state);
  }
  double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
  double next_double_open() { return double((next_u64() >> 11) + 1) * 0x1.0p-53; }
  double next_gaussian() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = next_double_open();
    const double u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(theta);
    have_spare = true;
    return r * std::cos(theta);
  }
};

inline int nthreads_or_default(int n) {
#ifdef _OPENMP
  return n > 0 ? n : omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

// fp64 dot product of two fp32 rows, fixed 8-lane order (see header comment).
inline double dot_f32(const float* a, const float* b, int d) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= d; c += 8)
    for (int l = 0; l < 8; ++l) acc[l] += double(a[c + l]) * double(b[c + l]);
  for (int l = 0; c < d; ++c, ++l) acc[l] += double(a[c]) * double(b[c]);
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}
inline double dot_f64(const double* a, const float* b, int d) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= d; c += 8)
    for (int l = 0; l < 8; ++l) acc[l] += a[c + l] * double(b[c + l]);
  for (int l = 0; c < d; ++c, ++l) acc[l] += a[c] * double(b[c]);
  return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// sample_distinct (workloads.cpp:37-46): partial Fisher-Yates, then sort.
std::vector<int> sample_distinct(Rng& rng, std::vector<int> pool, int m_take) {
  for (int t = 0; t < m_take; ++t) {
    const int swap_with = t + int(rng.next_u64() % uint64_t(pool.size() - t));
    std::swap(pool[t], pool[swap_with]);
  }
  pool.resize(m_take);
  std::sort(pool.begin(), pool.end());
  return pool;
}

// stable descending order, ties by ascending index (selection.cpp:20-23).
std::vector<int> argsort_desc(const double* v, int n) {
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return v[a] > v[b]; });
  return order;
}

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }

uint64_t or_mix64(uint64_t z) { return mix64(z); }
uint64_t or_chain_seed(uint64_t seed, uint64_t tag) { return chain(seed, tag); }

void or_rng_draws(uint64_t stream_seed, int kind, int n, uint64_t* out) {
  Rng rng(stream_seed);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = rng.next_u64();
      continue;
    }
    double v = kind == 1 ? rng.next_double() : kind == 2 ? rng.next_double_open() : rng.next_gaussian();
    std::memcpy(&out[i], &v, 8);
  }
}

// gen_workload (workloads.cpp:66-128). GQA extension: K/V noise streams are
// per KV head g (role tags 1/2, head g); planted directions of Q head h are
// added to K head h / (H/H_kv) in (h, i, j) order. H_kv == H reproduces the
// reference generator exactly.
int or_gen_workload(int kind, int L, int H, int H_kv, int d_k, int S, uint64_t seed,
                    double sigma, double gain_d, int m, float* Q, float* K, float* V,
                    int32_t* planted, int nthreads) {
  if (L <= 0 || H <= 0 || d_k <= 0 || S <= 0 || L % S != 0)
    return fail("gen_workload: need positive dims with L divisible by S");
  if (H_kv <= 0 || H % H_kv != 0) return fail("gen_workload: H must be a multiple of H_kv");
  const int N = L / S;
  const bool planted_kind = kind != OR_WL_GAUSSIAN;
  if (planted_kind) {
    if (m < 1 || m > N) return fail("gen_workload: m must lie in [1, N]");
    if (kind == OR_WL_LOCALITY_SHIFT && (N < 2 || m > N - N / 2))
      return fail("gen_workload: locality_shift needs m plantable in the upper half of blocks");
    if (!(sigma > 0.0) || !(gain_d >= 0.0))
      return fail("gen_workload: sigma must be positive, gain nonnegative");
  }
  const double scale = planted_kind ? sigma : 1.0;
  const int nt = nthreads_or_default(nthreads);
  // noise: gaussian_stack (workloads.cpp:18-26), one stream per (role, head, block)
  struct Job { int role, h, b; };
  std::vector<Job> jobs;
  for (int h = 0; h < H; ++h)
    for (int b = 0; b < N; ++b) jobs.push_back({0, h, b});
  for (int role = 1; role <= 2; ++role)
    for (int h = 0; h < H_kv; ++h)
      for (int b = 0; b < N; ++b) jobs.push_back({role, h, b});
#pragma omp parallel for schedule(dynamic, 16) num_threads(nt)
  for (long long jj = 0; jj < (long long)jobs.size(); ++jj) {
    const Job jb = jobs[jj];
    float* base = jb.role == 0 ? Q : jb.role == 1 ? K : V;
    float* m0 = base + (size_t(jb.h) * L + size_t(jb.b) * S) * d_k;
    Rng rng(chain(seed, uint64_t(jb.role), uint64_t(jb.h), uint64_t(jb.b)));
    for (int r = 0; r < S; ++r)
      for (int c = 0; c < d_k; ++c) m0[size_t(r) * d_k + c] = float(scale * rng.next_gaussian());
  }
  if (planted)
    for (size_t t = 0; t < size_t(H) * N * (planted_kind ? m : 1); ++t) planted[t] = -1;
  if (!planted_kind) return 0;

  const float gain = float(gain_d);
  const int G = H / H_kv;
  for (int h = 0; h < H; ++h) {
    const int g = h / G;
    std::vector<int> last_set;
    if (kind == OR_WL_LOCALITY_SHIFT) {
      Rng rng(chain(seed, 3, uint64_t(h), uint64_t(N - 1)));
      std::vector<int> upper;
      for (int j = N / 2; j < N; ++j) upper.push_back(j);
      last_set = sample_distinct(rng, upper, m);
    }
    for (int i = 0; i < N; ++i) {
      std::vector<int> set;
      if (kind == OR_WL_LOCALITY_SHIFT && i == N - 1) {
        set = last_set;
      } else {
        Rng rng(chain(seed, 3, uint64_t(h), uint64_t(i)));
        std::vector<int> pool;
        for (int j = 0; j <= i; ++j)
          if (kind != OR_WL_LOCALITY_SHIFT ||
              !std::binary_search(last_set.begin(), last_set.end(), j))
            pool.push_back(j);
        set = sample_distinct(rng, pool, std::min(m, int(pool.size())));
      }
      Rng dir_rng(chain(seed, 4, uint64_t(h), uint64_t(i)));
      std::vector<double> u(d_k);
      for (int c = 0; c < d_k; ++c) u[c] = dir_rng.next_gaussian();
      double n2 = 0.0;
      for (int c = 0; c < d_k; ++c) n2 += u[c] * u[c];
      const double n = std::sqrt(n2);
      if (n > 0.0)
        for (int c = 0; c < d_k; ++c) u[c] /= n;
      std::vector<float> gu(d_k);
      for (int c = 0; c < d_k; ++c) gu[c] = gain * float(u[c]);
      for (int r = i * S; r < (i + 1) * S; ++r)
        for (int c = 0; c < d_k; ++c) Q[(size_t(h) * L + r) * d_k + c] += gu[c];
      for (int j : set)
        for (int r = j * S; r < (j + 1) * S; ++r)
          for (int c = 0; c < d_k; ++c) K[(size_t(g) * L + r) * d_k + c] += gu[c];
      if (planted)
        for (size_t t = 0; t < set.size(); ++t) planted[(size_t(h) * N + i) * m + t] = set[t];
    }
  }
  return 0;
}

// validate_inputs (types.cpp:97-123) on flat shapes; GQA additions appended.
int or_validate(const or_cfg* c, char* msg, int cap) {
  std::vector<std::string> e;
  if (c->H <= 0) e.push_back("H must be positive");
  if (c->L <= 0) e.push_back("L must be positive");
  if (c->d_k <= 0) e.push_back("d_k must be positive");
  if (c->S <= 0) e.push_back("S must be positive");
  if (c->L > 0 && c->S > 0 && c->L % c->S != 0)
    e.push_back("L=" + std::to_string(c->L) + " not divisible by S=" + std::to_string(c->S));
  if (c->c_q <= 0) e.push_back("c_q must be positive");
  if (c->c_k <= 0) e.push_back("c_k must be positive");
  if (c->c_h <= 0) e.push_back("c_h must be positive");
  if (c->S > 0 && c->c_q > 0 && c->S % c->c_q != 0)
    e.push_back("S=" + std::to_string(c->S) + " not divisible by c_q=" + std::to_string(c->c_q));
  if (c->S > 0 && c->c_k > 0 && c->S % c->c_k != 0)
    e.push_back("S=" + std::to_string(c->S) + " not divisible by c_k=" + std::to_string(c->c_k));
  if (c->H > 0 && c->c_h > 0 && c->H % c->c_h != 0)
    e.push_back("H=" + std::to_string(c->H) + " not divisible by c_h=" + std::to_string(c->c_h));
  if (!(c->P > 0.0) || c->P > 1.0) e.push_back("P must lie in (0, 1]");
  if (c->H_kv <= 0) e.push_back("H_kv must be positive");
  if (c->H > 0 && c->H_kv > 0 && c->H % c->H_kv != 0)
    e.push_back("H=" + std::to_string(c->H) + " not divisible by H_kv=" + std::to_string(c->H_kv));
  std::string j;
  for (size_t i = 0; i < e.size(); ++i) j += (i ? "; " : "") + e[i];
  if (msg && cap > 0) std::snprintf(msg, size_t(cap), "%s", j.c_str());
  return int(e.size());
}

// pool_sequence (compression.hpp:13-57)
int or_pool_sequence(const float* x, int rows, int cols, int c, int strategy, uint64_t seed,
                     float* out) {
  if (c <= 0) return fail("pool_sequence: c must be positive");
  if (rows % c != 0)
    return fail("pool_sequence: rows (" + std::to_string(rows) + ") not divisible by c (" +
                std::to_string(c) + ")");
  if (c == 1) {
    std::memcpy(out, x, sizeof(float) * size_t(rows) * cols);
    return 0;
  }
  const int out_rows = rows / c;
  for (int w = 0; w < out_rows; ++w) {
    const float* win = x + size_t(w) * c * cols;
    float* o = out + size_t(w) * cols;
    if (strategy == OR_POOL_MEAN) {
      for (int col = 0; col < cols; ++col) {
        double acc = 0.0;
        for (int r = 0; r < c; ++r) acc += double(win[size_t(r) * cols + col]);
        o[col] = float(acc / double(c));
      }
    } else if (strategy == OR_POOL_MAX) {
      for (int col = 0; col < cols; ++col) {
        float best = win[col];
        for (int r = 1; r < c; ++r) best = std::max(best, win[size_t(r) * cols + col]);
        o[col] = best;
      }
    } else {
      Rng rng(chain(seed, uint64_t(w)));
      std::vector<double> norms(c);
      double total = 0.0;
      for (int r = 0; r < c; ++r) {
        double s2 = 0.0;
        for (int col = 0; col < cols; ++col) {
          const double v = double(win[size_t(r) * cols + col]);
          s2 += v * v;
        }
        norms[r] = std::sqrt(s2);
      }
      for (int r = 0; r < c; ++r) total += norms[r];
      int pick = c - 1;
      if (total > 0.0) {
        const double u = rng.next_double() * total;
        double cum = 0.0;
        for (int r = 0; r < c; ++r) {
          cum += norms[r];
          if (u < cum) {
            pick = r;
            break;
          }
        }
      } else {
        pick = int(rng.next_u64() % uint64_t(c));
      }
      std::memcpy(o, win + size_t(pick) * cols, sizeof(float) * cols);
    }
  }
  return 0;
}

// compress (compression.cpp:5-25) with pool_heads (compression.hpp:61-76).
int or_compress(const or_cfg* cfg, const float* Q, const float* K, float* Qc, float* Kc) {
  char msg[1024];
  if (or_validate(cfg, msg, sizeof msg)) return fail(std::string("compress: ") + msg);
  const int H = cfg->H, L = cfg->L, d = cfg->d_k, G = H / cfg->H_kv, ch = cfg->c_h;
  const int Lq = L / cfg->c_q, Lk = L / cfg->c_k;
  std::vector<float> qs(size_t(Lq) * d), ks(size_t(Lk) * d);
  std::vector<double> qacc(size_t(Lq) * d), kacc(size_t(Lk) * d);
  for (int hc = 0; hc < H / ch; ++hc) {
    for (int g = 0; g < ch; ++g) {
      const int h = hc * ch + g;
      int rc = or_pool_sequence(Q + size_t(h) * L * d, L, d, cfg->c_q, cfg->strategy,
                                chain(cfg->seed, 0, uint64_t(h)), qs.data());
      rc |= or_pool_sequence(K + size_t(h / G) * L * d, L, d, cfg->c_k, cfg->strategy,
                             chain(cfg->seed, 1, uint64_t(h)), ks.data());
      if (rc) return rc;
      if (ch == 1) {
        std::memcpy(Qc + size_t(hc) * Lq * d, qs.data(), sizeof(float) * qs.size());
        std::memcpy(Kc + size_t(hc) * Lk * d, ks.data(), sizeof(float) * ks.size());
        continue;
      }
      for (size_t t = 0; t < qs.size(); ++t) qacc[t] = g == 0 ? double(qs[t]) : qacc[t] + double(qs[t]);
      for (size_t t = 0; t < ks.size(); ++t) kacc[t] = g == 0 ? double(ks[t]) : kacc[t] + double(ks[t]);
    }
    if (ch > 1) {
      for (size_t t = 0; t < qacc.size(); ++t) Qc[size_t(hc) * Lq * d + t] = float(qacc[t] / double(ch));
      for (size_t t = 0; t < kacc.size(); ++t) Kc[size_t(hc) * Lk * d + t] = float(kacc[t] / double(ch));
    }
  }
  return 0;
}

namespace {
// One composite query row: softmax over live composite keys (proxy.cpp:28-42),
// then region sums accumulated into score_row[j] for j <= i (proxy.cpp:60-66).
void proxy_row(const or_cfg* cfg, const float* q, const float* Kc, int Lk, int t,
               std::vector<double>& logits, double* A_row) {
  const int d = cfg->d_k;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  for (int s = 0; s < Lk; ++s) logits[s] = dot_f32(q, Kc + size_t(s) * d, d) * inv_scale;
  int live = Lk;
  if (cfg->causal_mode == OR_PRE_SOFTMAX) {
    const int64_t last_q = int64_t(t + 1) * cfg->c_q - 1;
    live = std::min<int64_t>(live, last_q / cfg->c_k + 1);
  }
  double m = logits[0];
  for (int s = 1; s < live; ++s) m = std::max(m, logits[s]);
  double den = 0.0;
  for (int s = 0; s < live; ++s) {
    logits[s] = std::exp(logits[s] - m);
    den += logits[s];
  }
  for (int s = 0; s < live; ++s) A_row[s] = logits[s] / den;
  for (int s = live; s < Lk; ++s) A_row[s] = 0.0;
}

void proxy_block_row(const or_cfg* cfg, const float* Qc_h, const float* Kc_h, int i,
                     double* score_row, double* A_out_h) {
  const int S = cfg->S, N = cfg->L / S, Lk = cfg->L / cfg->c_k, d = cfg->d_k;
  const int rq = S / cfg->c_q, rk = S / cfg->c_k;
  std::vector<double> logits(Lk), A(size_t(rq) * Lk);
  for (int r = 0; r < rq; ++r) {
    const int t = i * rq + r;
    proxy_row(cfg, Qc_h + size_t(t) * d, Kc_h, Lk, t, logits, A.data() + size_t(r) * Lk);
  }
  if (A_out_h) std::memcpy(A_out_h + size_t(i) * rq * Lk, A.data(), sizeof(double) * A.size());
  for (int j = 0; j < N; ++j) {
    if (j > i) {
      score_row[j] = kMaskedScore;
      continue;
    }
    double sum = 0.0;
    for (int r = 0; r < rq; ++r)
      for (int s = j * rk; s < (j + 1) * rk; ++s) sum += A[size_t(r) * Lk + s];
    score_row[j] = sum;
  }
}
}  // namespace

int or_proxy_scores(const or_cfg* cfg, const float* Qc, const float* Kc, double* scores,
                    double* A_out, int nthreads) {
  char msg[1024];
  if (or_validate(cfg, msg, sizeof msg)) return fail(std::string("proxy_scores: ") + msg);
  const int Hc = cfg->H / cfg->c_h, N = cfg->L / cfg->S, d = cfg->d_k;
  const int Lq = cfg->L / cfg->c_q, Lk = cfg->L / cfg->c_k;
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nt)
  for (int hc = 0; hc < Hc; ++hc)
    for (int i = 0; i < N; ++i)
      proxy_block_row(cfg, Qc + size_t(hc) * Lq * d, Kc + size_t(hc) * Lk * d, i,
                      scores + (size_t(hc) * N + i) * N,
                      A_out ? A_out + size_t(hc) * Lq * Lk : nullptr);
  return 0;
}

int or_proxy_score_rows(const or_cfg* cfg, const float* Qc, const float* Kc, int hc,
                        const int32_t* qblocks, int nrows, double* out, int nthreads) {
  const int N = cfg->L / cfg->S, d = cfg->d_k;
  const int Lq = cfg->L / cfg->c_q, Lk = cfg->L / cfg->c_k;
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int r = 0; r < nrows; ++r)
    proxy_block_row(cfg, Qc + size_t(hc) * Lq * d, Kc + size_t(hc) * Lk * d, qblocks[r],
                    out + size_t(r) * N, nullptr);
  return 0;
}

// antidiagonal_block_scores (baselines.cpp:10-52): every query t samples the keys
// s = res, res + stride, ... <= t with res = (S - 1 - t % S) % stride, softmax over
// those samples, probabilities added to score(t / S, s / S); j > i masked.
int or_antidiagonal_block_scores(int H, int H_kv, int L, int d, int S, int stride, const float* Q,
                                 const float* K, double* scores, int nthreads) {
  if (H <= 0 || L <= 0 || d <= 0 || S <= 0 || L % S || H_kv <= 0 || H % H_kv)
    return fail("antidiagonal_block_scores: bad dimensions");
  if (stride <= 0 || S % stride != 0) return fail("antidiagonal_block_scores: stride must divide S");
  const int N = L / S, G = H / H_kv;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nt)
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      const float* Kh = K + size_t(h / G) * L * d;
      double* row = scores + (size_t(h) * N + i) * N;
      for (int j = 0; j < N; ++j) row[j] = j <= i ? 0.0 : kMaskedScore;
      std::vector<double> logits;
      for (int q = 0; q < S; ++q) {
        const int t = i * S + q;
        const int res = (S - 1 - q) % stride;
        if (res > t) continue;
        const int cnt = (t - res) / stride + 1;
        logits.resize(cnt);
        const float* qt = Q + (size_t(h) * L + t) * d;
        double m = -kInf;
        for (int c = 0; c < cnt; ++c) {
          logits[c] = dot_f32(qt, Kh + size_t(res + c * stride) * d, d) * inv_scale;
          m = std::max(m, logits[c]);
        }
        double den = 0.0;
        for (int c = 0; c < cnt; ++c) {
          logits[c] = std::exp(logits[c] - m);
          den += logits[c];
        }
        for (int c = 0; c < cnt; ++c) row[(res + c * stride) / S] += logits[c] / den;
      }
    }
  return 0;
}

// last_block_probe_scores (baselines.cpp:54-87): column mass of the last S query
// rows (causal), replicated to every row's causal prefix.
int or_last_block_probe_scores(int H, int H_kv, int L, int d, int S, const float* Q, const float* K,
                               double* scores, int nthreads) {
  if (H <= 0 || L <= 0 || d <= 0 || S <= 0 || L % S || H_kv <= 0 || H % H_kv)
    return fail("last_block_probe_scores: bad dimensions");
  const int N = L / S, G = H / H_kv;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int h = 0; h < H; ++h) {
    const float* Kh = K + size_t(h / G) * L * d;
    std::vector<double> colmass(N, 0.0), row(L);
    for (int r = 0; r < S; ++r) {
      const float* qt = Q + (size_t(h) * L + size_t(N - 1) * S + r) * d;
      const int live = (N - 1) * S + r + 1;
      double m = -kInf;
      for (int k = 0; k < live; ++k) {
        row[k] = dot_f32(qt, Kh + size_t(k) * d, d) * inv_scale;
        m = std::max(m, row[k]);
      }
      double den = 0.0;
      for (int k = 0; k < live; ++k) {
        row[k] = std::exp(row[k] - m);
        den += row[k];
      }
      for (int j = 0; j < N; ++j) {
        const int len = std::min(S, live - j * S);
        if (len <= 0) continue;
        double seg = 0.0;
        for (int k = 0; k < len; ++k) seg += row[j * S + k];
        colmass[j] += seg / den;
      }
    }
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) scores[(size_t(h) * N + i) * N + j] = j <= i ? colmass[j] : kMaskedScore;
  }
  return 0;
}

// top_p_row (selection.cpp:11-48)
int or_top_p_row(const double* scores, int n, double P, int32_t* indices, int* count,
                 double* covered) {
  if (n <= 0) return fail("top_p_row: empty score row");
  if (!(P > 0.0) || P > 1.0) return fail("top_p_row: P must lie in (0, 1]");
  for (int i = 0; i < n; ++i)
    if (!(scores[i] >= 0.0)) return fail("top_p_row: scores must be nonnegative");
  const std::vector<int> order = argsort_desc(scores, n);
  double total = 0.0;
  for (int idx : order) total += scores[idx];
  if (total <= 0.0) {
    indices[0] = n - 1;
    *count = 1;
    *covered = 1.0;
    return 0;
  }
  if (P >= 1.0) {
    for (int t = 0; t < n; ++t) indices[t] = order[t];
    *count = n;
    *covered = 1.0;
    return 0;
  }
  double cum = 0.0;
  int k = 0;
  for (int idx : order) {
    indices[k++] = idx;
    cum += scores[idx];
    if (cum >= P * total) break;
  }
  *count = k;
  *covered = cum / total;
  return 0;
}

// top-k extension (not in the reference): the first min(k, n)
// entries of the same stable order; covered = their sequential mass / total.
int or_top_k_row(const double* scores, int n, int k, int32_t* indices, int* count,
                 double* covered) {
  if (n <= 0) return fail("top_k_row: empty score row");
  if (k < 1) return fail("top_k_row: k must be positive");
  for (int i = 0; i < n; ++i)
    if (!(scores[i] >= 0.0)) return fail("top_k_row: scores must be nonnegative");
  const std::vector<int> order = argsort_desc(scores, n);
  double total = 0.0;
  for (int idx : order) total += scores[idx];
  const int kk = std::min(k, n);
  double cum = 0.0;
  for (int t = 0; t < kk; ++t) {
    indices[t] = order[t];
    cum += scores[order[t]];
  }
  *count = kk;
  *covered = total > 0.0 ? cum / total : 1.0;
  return 0;
}

// build_block_mask (selection.cpp:60-88)
int or_build_block_mask(const double* scores, int H, int N, int c_h, int select_mode, double P,
                        int top_k, uint8_t* mask, double* coverage) {
  if (c_h <= 0 || H <= 0) return fail("build_block_mask: c_h and H must be positive");
  if (H % c_h != 0) return fail("build_block_mask: H not divisible by c_h");
  std::memset(mask, 0, size_t(H) * N * N);
  std::vector<int32_t> idx(N);
  for (int hc = 0; hc < H / c_h; ++hc)
    for (int i = 0; i < N; ++i) {
      const double* row = scores + (size_t(hc) * N + i) * N;
      int cnt = 0;
      double cov = 0.0;
      const int rc = select_mode == OR_SELECT_TOP_K
                         ? or_top_k_row(row, i + 1, top_k, idx.data(), &cnt, &cov)
                         : or_top_p_row(row, i + 1, P, idx.data(), &cnt, &cov);
      if (rc) return rc;
      for (int g = 0; g < c_h; ++g) {
        const int h = hc * c_h + g;
        for (int t = 0; t < cnt; ++t) mask[(size_t(h) * N + i) * N + idx[t]] = 1;
        coverage[size_t(h) * N + i] = cov;
      }
    }
  return 0;
}

// dense_attention (attention.cpp:20-54); masked (future) entries contribute
// exact zeros in the reference, so only the live prefix is computed here.
int or_dense_attention(int H, int H_kv, int L, int d, const float* Q, const float* K,
                       const float* V, int causal, float* O, double* lse, int nthreads) {
  if (H <= 0 || L <= 0 || d <= 0 || H_kv <= 0 || H % H_kv)
    return fail("dense_attention: bad dimensions");
  const int G = H / H_kv;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 8) num_threads(nt)
  for (int h = 0; h < H; ++h)
    for (int t = 0; t < L; ++t) {
      const float* Kh = K + size_t(h / G) * L * d;
      const float* Vh = V + size_t(h / G) * L * d;
      const float* q = Q + (size_t(h) * L + t) * d;
      const int live = causal ? t + 1 : L;
      std::vector<double> p(live), acc(d, 0.0);
      double m = -kInf;
      for (int k = 0; k < live; ++k) {
        p[k] = dot_f32(q, Kh + size_t(k) * d, d) * inv_scale;
        m = std::max(m, p[k]);
      }
      double den = 0.0;
      for (int k = 0; k < live; ++k) {
        p[k] = std::exp(p[k] - m);
        den += p[k];
      }
      for (int k = 0; k < live; ++k) p[k] /= den;
      for (int k = 0; k < live; ++k) {
        const float* v = Vh + size_t(k) * d;
        for (int c = 0; c < d; ++c) acc[c] += p[k] * double(v[c]);
      }
      for (int c = 0; c < d; ++c) O[(size_t(h) * L + t) * d + c] = float(acc[c]);
      if (lse) lse[size_t(h) * L + t] = m + std::log(den);
    }
  return 0;
}

// exact_block_mass (attention.cpp:56-87)
int or_exact_block_mass(int H, int H_kv, int L, int d, int S, const float* Q, const float* K,
                        double* mass, int nthreads) {
  if (H <= 0 || L <= 0 || d <= 0 || S <= 0 || L % S || H_kv <= 0 || H % H_kv)
    return fail("exact_block_mass: bad dimensions");
  const int N = L / S, G = H / H_kv;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  const int nt = nthreads_or_default(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nt)
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      const float* Kh = K + size_t(h / G) * L * d;
      double* row = mass + (size_t(h) * N + i) * N;
      for (int j = 0; j < N; ++j) row[j] = j <= i ? 0.0 : kMaskedScore;
      std::vector<double> p(size_t(i + 1) * S);
      for (int r = 0; r < S; ++r) {
        const float* q = Q + (size_t(h) * L + size_t(i) * S + r) * d;
        const int live = i * S + r + 1;
        double m = -kInf;
        for (int k = 0; k < live; ++k) {
          p[k] = dot_f32(q, Kh + size_t(k) * d, d) * inv_scale;
          m = std::max(m, p[k]);
        }
        double den = 0.0;
        for (int k = 0; k < live; ++k) {
          p[k] = std::exp(p[k] - m);
          den += p[k];
        }
        for (int j = 0; j <= i; ++j) {
          const int k0 = j * S, len = std::min(S, live - k0);
          if (len <= 0) continue;
          double seg = 0.0;
          for (int k = k0; k < k0 + len; ++k) seg += p[k];
          row[j] += seg / den;
        }
      }
    }
  return 0;
}

namespace {
// One (head, query block) of block_sparse_attention (attention.cpp:99-135).
int sparse_block(int L, int d, int S, const float* Qh, const float* Kh, const float* Vh,
                 const uint8_t* mrow, int i, float* O, double* lse) {
  const int N = L / S;
  const double inv_scale = 1.0 / std::sqrt(double(d));
  for (int j = i + 1; j < N; ++j)
    if (mrow[j]) return 1;
  std::vector<double> qd(size_t(S) * d), m(S, -kInf), den(S, 0.0), acc(size_t(S) * d, 0.0);
  std::vector<double> tile(size_t(S) * S), pv(size_t(S) * d), scale(S);
  for (size_t t = 0; t < qd.size(); ++t) qd[t] = double(Qh[size_t(i) * S * d + t]);
  bool any = false;
  for (int j = 0; j <= i; ++j) {
    if (!mrow[j]) continue;
    any = true;
    for (int r = 0; r < S; ++r)
      for (int c = 0; c < S; ++c)
        tile[size_t(r) * S + c] =
            dot_f64(&qd[size_t(r) * d], Kh + (size_t(j) * S + c) * d, d) * inv_scale;
    if (j == i)
      for (int r = 0; r + 1 < S; ++r)
        for (int c = r + 1; c < S; ++c) tile[size_t(r) * S + c] = -kInf;
    for (int r = 0; r < S; ++r) {
      double rmax = tile[size_t(r) * S];
      for (int c = 1; c < S; ++c) rmax = std::max(rmax, tile[size_t(r) * S + c]);
      const double m_new = std::max(m[r], rmax);
      scale[r] = den[r] == 0.0 ? 0.0 : std::exp(m[r] - m_new);
      double rs = 0.0;
      for (int c = 0; c < S; ++c) {
        const double e = std::exp(tile[size_t(r) * S + c] - m_new);
        tile[size_t(r) * S + c] = e;
        rs += e;
      }
      den[r] = den[r] * scale[r] + rs;
      m[r] = m_new;
    }
    std::fill(pv.begin(), pv.end(), 0.0);
    for (int r = 0; r < S; ++r)
      for (int k = 0; k < S; ++k) {
        const double e = tile[size_t(r) * S + k];
        const float* v = Vh + (size_t(j) * S + k) * d;
        double* o = &pv[size_t(r) * d];
        for (int c = 0; c < d; ++c) o[c] += e * double(v[c]);
      }
    for (int r = 0; r < S; ++r)
      for (int c = 0; c < d; ++c)
        acc[size_t(r) * d + c] = acc[size_t(r) * d + c] * scale[r] + pv[size_t(r) * d + c];
  }
  if (!any) return 2;
  for (int r = 0; r < S; ++r) {
    for (int c = 0; c < d; ++c) O[size_t(r) * d + c] = float(acc[size_t(r) * d + c] / den[r]);
    if (lse) lse[r] = m[r] + std::log(den[r]);
  }
  return 0;
}
}  // namespace

int or_block_sparse_attention(int H, int H_kv, int L, int d, int S, const float* Q,
                              const float* K, const float* V, const uint8_t* mask, float* O,
                              double* lse, int nthreads) {
  if (H <= 0 || L <= 0 || d <= 0 || S <= 0 || L % S || H_kv <= 0 || H % H_kv)
    return fail("block_sparse_attention: bad dimensions");
  const int N = L / S, G = H / H_kv;
  const int nt = nthreads_or_default(nthreads);
  std::vector<int> status(size_t(H) * N, 0);
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(nt)
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i)
      status[size_t(h) * N + i] = sparse_block(
          L, d, S, Q + size_t(h) * L * d, K + size_t(h / G) * L * d, V + size_t(h / G) * L * d,
          mask + (size_t(h) * N + i) * N, i, O + (size_t(h) * L + size_t(i) * S) * d,
          lse ? lse + size_t(h) * L + size_t(i) * S : nullptr);
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      const int s = status[size_t(h) * N + i];
      if (s == 1) return fail("block_sparse_attention: mask selects a non-causal block");
      if (s == 2)
        return fail("block_sparse_attention: query block " + std::to_string(i) +
                    " has no selected key block");
    }
  return 0;
}

int or_block_sparse_attention_rows(int H, int H_kv, int L, int d, int S, const float* Q,
                                   const float* K, const float* V, const uint8_t* mask,
                                   const int32_t* heads, const int32_t* qblocks, int nrows,
                                   float* O, double* lse, int nthreads) {
  const int N = L / S, G = H / H_kv;
  const int nt = nthreads_or_default(nthreads);
  std::vector<int> status(nrows, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int r = 0; r < nrows; ++r) {
    const int h = heads[r], i = qblocks[r];
    status[r] = sparse_block(L, d, S, Q + size_t(h) * L * d, K + size_t(h / G) * L * d,
                             V + size_t(h / G) * L * d, mask + (size_t(h) * N + i) * N, i,
                             O + size_t(r) * S * d, lse ? lse + size_t(r) * S : nullptr);
  }
  for (int r = 0; r < nrows; ++r)
    if (status[r]) return fail("block_sparse_attention_rows: invalid mask row");
  return 0;
}

namespace {
uint64_t ceil_log2(uint64_t n) {
  uint64_t bits = 0;
  while ((uint64_t(1) << bits) < n) ++bits;
  return bits;
}
}  // namespace

// selection_flops (metrics.cpp:44-81)
int or_selection_flops(uint64_t L, uint64_t H, uint64_t d, uint64_t S, int c_q, int c_k, int c_h,
                       int proxy, uint64_t stride, uint64_t* f) {
  if (L == 0 || H == 0 || d == 0 || S == 0 || L % S != 0)
    return fail("selection_flops: bad dimensions");
  const uint64_t N = L / S;
  for (int t = 0; t < 6; ++t) f[t] = 0;
  f[5] = 4 * L * L * H * d;
  if (proxy == OR_PROXY_UNISPARSE) {
    const uint64_t cq = uint64_t(c_q), ck = uint64_t(c_k), ch = uint64_t(c_h);
    if (c_q <= 0 || c_k <= 0 || c_h <= 0 || S % cq != 0 || S % ck != 0 || H % ch != 0)
      return fail("selection_flops: bad compression factors");
    f[0] = 2 * L * H * d;
    if (ch > 1) f[0] += 2 * (L / cq + L / ck) * H * d;
    f[1] = 2 * (L / cq) * (L / ck) * (H / ch) * d;
    f[2] = 4 * (L / cq) * (L / ck) * (H / ch);
    f[3] = (H / ch) * N * N * ceil_log2(N);
  } else if (proxy == OR_PROXY_ANTIDIAGONAL) {
    if (stride == 0 || S % stride != 0) return fail("selection_flops: stride must divide S");
    f[1] = 2 * L * (L / stride) * H * d;
    f[2] = 2 * L * (L / stride) * H;
    f[3] = H * N * N * ceil_log2(N);
  } else {
    f[1] = 2 * S * L * H * d;
    f[2] = 2 * S * L * H;
    f[3] = H * N * N * ceil_log2(N);
  }
  return 0;
}

// output_fidelity (metrics.cpp:118-151)
int or_output_fidelity(const float* test, const float* ref, int H, int L, int d, double* out3) {
  double max_abs = 0.0, rel_sum = 0.0, cos_sum = 0.0;
  int64_t entries = 0, rows = 0;
  for (int64_t r = 0; r < int64_t(H) * L; ++r) {
    double dot = 0.0, nt = 0.0, nr = 0.0;
    for (int c = 0; c < d; ++c) {
      const double t = test[r * d + c], rf = ref[r * d + c];
      const double df = std::abs(t - rf);
      max_abs = std::max(max_abs, df);
      rel_sum += df / std::max(std::abs(rf), 1e-6);
      ++entries;
      dot += t * rf;
      nt += t * t;
      nr += rf * rf;
    }
    if (nt == 0.0 && nr == 0.0)
      cos_sum += 1.0;
    else if (nt == 0.0 || nr == 0.0)
      cos_sum += 0.0;
    else
      cos_sum += dot / std::sqrt(nt * nr);
    ++rows;
  }
  out3[0] = max_abs;
  out3[1] = rel_sum / double(entries);
  out3[2] = cos_sum / double(rows);
  return 0;
}

// argsort_desc / average_ranks (metrics.cpp:17-40): stable orders, average ranks for ties.
static std::vector<int> argsort_desc_or(const double* v, int n) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return v[a] > v[b]; });
  return order;
}
static std::vector<double> average_ranks_or(const double* v, int n) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return v[a] < v[b]; });
  std::vector<double> ranks(n);
  int i = 0;
  while (i < n) {
    int j = i;
    while (j + 1 < n && v[order[j + 1]] == v[order[i]]) ++j;
    const double r = 0.5 * (i + j) + 1.0;
    for (int t = i; t <= j; ++t) ranks[order[t]] = r;
    i = j + 1;
  }
  return ranks;
}

// spearman_rho (metrics.cpp:100-116); returns 0 and sets *defined = 0 for a flat side.
int or_spearman_rho(const double* a, const double* b, int n, double* rho, int* defined) {
  if (n < 2) return fail("spearman_rho: need at least 2 values");
  const auto ra = average_ranks_or(a, n), rb = average_ranks_or(b, n);
  const double mean = (double(n) + 1.0) / 2.0;
  double va = 0.0, vb = 0.0, cov = 0.0;
  for (int i = 0; i < n; ++i) {
    const double da = ra[i] - mean, db = rb[i] - mean;
    va += da * da;
    vb += db * db;
    cov += da * db;
  }
  *defined = !(va == 0.0 || vb == 0.0);
  *rho = *defined ? cov / std::sqrt(va * vb) : 0.0;
  return 0;
}

// block_recall (metrics.cpp:155-176): mask [H][N][N] bytes, reference scores [H][N][N].
int or_block_recall(const uint8_t* mask, const double* ref, int H, int N, int k, double* out) {
  if (k < 1 || k > N) return fail("block_recall: k out of range");
  double sum = 0.0;
  int64_t rows = 0;
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      const int k_eff = std::min(k, i + 1);
      const double* row = ref + (size_t(h) * N + i) * N;
      const auto order = argsort_desc_or(row, i + 1);
      int hit = 0;
      for (int t = 0; t < k_eff; ++t) hit += mask[(size_t(h) * N + i) * N + order[t]] ? 1 : 0;
      sum += double(hit) / double(k_eff);
      ++rows;
    }
  *out = sum / double(rows);
  return 0;
}

// planted_recall (metrics.cpp:178-199): mask [H][N][N] bytes, planted [H][N][m] (-1 = none).
int or_planted_recall(const uint8_t* mask, const int32_t* planted, int H, int N, int m, double* out) {
  double sum = 0.0;
  int64_t rows = 0;
  for (int h = 0; h < H; ++h)
    for (int i = 0; i < N; ++i) {
      int want = 0, hit = 0;
      for (int t = 0; t < m; ++t) {
        const int j = planted[(size_t(h) * N + i) * m + t];
        if (j < 0) continue;
        ++want;
        hit += mask[(size_t(h) * N + i) * N + j] ? 1 : 0;
      }
      if (want == 0) continue;
      sum += double(hit) / double(want);
      ++rows;
    }
  if (rows == 0) return fail("planted_recall: no planted rows");
  *out = sum / double(rows);
  return 0;
}

// mean_row_spearman (metrics.cpp:201-224): proxy [H/c_h][N][N], reference [H][N][N].
int or_mean_row_spearman(const double* proxy, const double* ref, int H, int N, int c_h, double* mean,
                         int64_t* defined, int64_t* undefined) {
  if (c_h <= 0 || H % c_h != 0) return fail("mean_row_spearman: head counts disagree");
  double sum = 0.0;
  int64_t d = 0, u = 0;
  for (int h = 0; h < H; ++h)
    for (int i = 1; i < N; ++i) {
      double rho;
      int def;
      or_spearman_rho(proxy + (size_t(h / c_h) * N + i) * N, ref + (size_t(h) * N + i) * N, i + 1, &rho, &def);
      if (def) {
        sum += rho;
        ++d;
      } else {
        ++u;
      }
    }
  *mean = d ? sum / double(d) : 0.0;
  *defined = d;
  *undefined = u;
  return 0;
}

// unisparse_attn (pipeline.cpp:19-24): compress -> proxy -> mask -> sparse attention.
int or_unisparse_attn(const or_cfg* cfg, const float* Q, const float* K, const float* V,
                      float* O, double* lse, uint8_t* mask, double* coverage, int nthreads) {
  char msg[1024];
  if (or_validate(cfg, msg, sizeof msg)) return fail(std::string("select_blocks: ") + msg);
  const int Hc = cfg->H / cfg->c_h, N = cfg->L / cfg->S, d = cfg->d_k;
  std::vector<float> Qc(size_t(Hc) * (cfg->L / cfg->c_q) * d), Kc(size_t(Hc) * (cfg->L / cfg->c_k) * d);
  std::vector<double> scores(size_t(Hc) * N * N);
  int rc = or_compress(cfg, Q, K, Qc.data(), Kc.data());
  if (!rc) rc = or_proxy_scores(cfg, Qc.data(), Kc.data(), scores.data(), nullptr, nthreads);
  if (!rc)
    rc = or_build_block_mask(scores.data(), cfg->H, N, cfg->c_h, cfg->select_mode, cfg->P,
                             cfg->top_k, mask, coverage);
  if (!rc)
    rc = or_block_sparse_attention(cfg->H, cfg->H_kv, cfg->L, d, cfg->S, Q, K, V, mask, O, lse,
                                   nthreads);
  return rc;
}

}  // extern "C"
