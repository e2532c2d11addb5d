// metrics.cu — the reference's quality metrics on GPU outputs (
// metrics.cpp:100-224, used by run_experiment, experiment.cpp:280-437).
//
//   output_fidelity  (metrics.cpp:118-153)  one thread per row, the reference's
//                    sequential column loop in fp64 (mul and add rounded
//                    separately, as the x86 reference: no FMA contraction)
//   block_recall     (metrics.cpp:155-176)  one CTA per (b, h, i): the first
//                    k_eff entries of the stable descending order of the
//                    reference row prefix, found by a 32-step radix select on
//                    order-preserving keys (ties resolved by ascending index),
//                    hits counted against the mask row
//   mean_row_spearman (metrics.cpp:201-224) one CTA per (b, h, i >= 1): both
//                    prefixes sorted (bitonic, 64-bit value|index keys = the
//                    reference stable_sort), tie groups get average ranks,
//                    then the reference's sequential fp64 sums
//
// Every per-row value lands in a workspace array; a single-thread kernel adds
// them in the reference's (h, i) order, so recall, spearman and cosine are
// bit-identical to the reference given the same inputs (mean_rel sums per row
// first: equal to the reference within fp64 rounding).
#include <cfloat>

#include "host_util.hpp"
#include "kernels.cuh"

namespace us {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxN = 4096;

__device__ __forceinline__ float bf16f(uint16_t b) { return __uint_as_float(uint32_t(b) << 16); }

// ---------------------------------------------------------------- output_fidelity
__global__ void fidelity_rows_kernel(long long rows, int d, const uint16_t* __restrict__ test,
                                     const uint16_t* __restrict__ ref, double* __restrict__ row_cos,
                                     double* __restrict__ row_rel, double* __restrict__ row_max) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const uint16_t* t = test + r * d;
  const uint16_t* f = ref + r * d;
  double dot = 0.0, nt = 0.0, nr = 0.0, rel = 0.0, mx = 0.0;
  for (int c = 0; c < d; ++c) {
    const double tv = bf16f(t[c]), rv = bf16f(f[c]);
    const double ad = fabs(__dadd_rn(tv, -rv));
    mx = fmax(mx, ad);
    rel = __dadd_rn(rel, ad / fmax(fabs(rv), 1e-6));
    dot = __dadd_rn(dot, __dmul_rn(tv, rv));
    nt = __dadd_rn(nt, __dmul_rn(tv, tv));
    nr = __dadd_rn(nr, __dmul_rn(rv, rv));
  }
  double cs;
  if (nt == 0.0 && nr == 0.0) cs = 1.0;
  else if (nt == 0.0 || nr == 0.0) cs = 0.0;
  else cs = dot / sqrt(__dmul_rn(nt, nr));
  row_cos[r] = cs;
  row_rel[r] = rel;
  row_max[r] = mx;
}

__global__ void fidelity_final_kernel(long long rows, int d, const double* row_cos, const double* row_rel,
                                      const double* row_max, double* out3) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0, rel = 0.0, cs = 0.0;
  for (long long r = 0; r < rows; ++r) {
    mx = fmax(mx, row_max[r]);
    rel = __dadd_rn(rel, row_rel[r]);
    cs = __dadd_rn(cs, row_cos[r]);
  }
  out3[0] = mx;
  out3[1] = rel / double(rows * d);
  out3[2] = cs / double(rows);
}

// ---------------------------------------------------------------- block helpers
// order-preserving u32 key of a float (larger float -> larger key)
__device__ __forceinline__ uint32_t fkey(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int block_sum(int v, int* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int s = 0;
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

// ---------------------------------------------------------------- block_recall
struct RecallArgs {
  int B, H, N, W, planes, heads_per_plane, k;
  const uint32_t* mask;  // [B][planes][N][W]
  const float* ref;      // [B][H][N][N]
  double* row_val;       // [B][H][N]
};

__global__ void __launch_bounds__(kThreads) recall_rows_kernel(const RecallArgs a) {
  __shared__ uint32_t key[kMaxN];
  __shared__ uint32_t mbits[kMaxN / 32];
  __shared__ int red[kThreads / 32];
  __shared__ int scan[kThreads];
  const int i = blockIdx.x % a.N;
  const int bh = blockIdx.x / a.N;
  const int b = bh / a.H, h = bh % a.H;
  const int n = i + 1;
  const int k_eff = min(a.k, n);
  const float* row = a.ref + ((long long)bh * a.N + i) * a.N;
  const uint32_t* mrow = a.mask + ((long long)(b * a.planes + h / a.heads_per_plane) * a.N + i) * a.W;
  for (int j = threadIdx.x; j < n; j += kThreads) key[j] = fkey(row[j]);
  for (int w = threadIdx.x; w < (n + 31) / 32; w += kThreads) mbits[w] = mrow[w];
  __syncthreads();
  // largest T with #{key >= T} >= k_eff: the k_eff-th largest key
  uint32_t T = 0;
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = T | (1u << bit);
    int c = 0;
    for (int j = threadIdx.x; j < n; j += kThreads) c += key[j] >= cand;
    if (block_sum(c, red) >= k_eff) T = cand;
  }
  // entries > T are in; of the entries == T, the first (k_eff - #greater) by index
  const int per = (n + kThreads - 1) / kThreads;
  const int j0 = threadIdx.x * per, j1 = min(n, j0 + per);
  int gt = 0, eq = 0, hit_gt = 0;
  for (int j = j0; j < j1; ++j) {
    const bool m = (mbits[j >> 5] >> (j & 31)) & 1u;
    gt += key[j] > T;
    eq += key[j] == T;
    hit_gt += (key[j] > T) && m;
  }
  const int n_gt = block_sum(gt, red);
  const int hits_gt = block_sum(hit_gt, red);
  // exclusive scan of the per-thread equal counts (ascending index order)
  scan[threadIdx.x] = eq;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {
    const int v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  const int need_eq = k_eff - n_gt;
  int before = scan[threadIdx.x] - eq, hit_eq = 0;
  for (int j = j0; j < j1; ++j) {
    if (key[j] != T) continue;
    if (before < need_eq && ((mbits[j >> 5] >> (j & 31)) & 1u)) ++hit_eq;
    ++before;
  }
  const int hits = hits_gt + block_sum(hit_eq, red);
  if (threadIdx.x == 0) a.row_val[(long long)bh * a.N + i] = double(hits) / double(k_eff);
}

__global__ void ordered_mean_kernel(long long rows, const double* v, const uint8_t* defined, double* out,
                                    long long* n_def) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  long long c = 0;
  for (long long r = 0; r < rows; ++r) {
    if (defined && !defined[r]) continue;
    s = __dadd_rn(s, v[r]);
    ++c;
  }
  out[0] = c ? s / double(c) : 0.0;
  if (n_def) *n_def = c;
}

// ---------------------------------------------------------------- mean_row_spearman
struct SpearmanArgs {
  int B, H, N, c_h;
  const float* proxy;  // [B][H/c_h][N][N]
  const float* ref;    // [B][H][N][N]
  double* row_val;     // [B][H][N]
  uint8_t* defined;    // [B][H][N]
};

// ascending bitonic sort of n2 (power of two) 64-bit keys in shared memory
__device__ void bitonic_sort(unsigned long long* k, int n2) {
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n2 / 2; t += kThreads) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long x = k[lo], y = k[hi];
        if ((x > y) == up) {
          k[lo] = y;
          k[hi] = x;
        }
      }
    }
  __syncthreads();
}

// average ranks (metrics.cpp:25-40) of row[0..n) into rank[] (by original index)
__device__ void average_ranks(const float* row, int n, unsigned long long* k, int* gstart, double* rank) {
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int j = threadIdx.x; j < n2; j += kThreads)
    k[j] = j < n ? ((unsigned long long)fkey(row[j]) << 32) | uint32_t(j) : ~0ull;
  bitonic_sort(k, n2);
  // tie-group start: max-scan of (t if value differs from t-1) — per-thread chunk + block scan
  const int per = (n + kThreads - 1) / kThreads;
  const int t0 = threadIdx.x * per, t1 = min(n, t0 + per);
  int run = -1;
  for (int t = t0; t < t1; ++t) {
    if (t == 0 || (k[t] >> 32) != (k[t - 1] >> 32)) run = t;
    gstart[t] = run;
  }
  __syncthreads();
  // propagate starts across chunks: a chunk without a start inherits the previous one's
  __shared__ int carry[kThreads];
  carry[threadIdx.x] = (t0 < t1) ? gstart[t1 - 1] : -1;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {
    const int v = threadIdx.x >= o ? carry[threadIdx.x - o] : -1;
    __syncthreads();
    carry[threadIdx.x] = max(carry[threadIdx.x], v);
    __syncthreads();
  }
  const int prev = threadIdx.x > 0 ? carry[threadIdx.x - 1] : -1;
  for (int t = t0; t < t1; ++t)
    if (gstart[t] < 0) gstart[t] = prev;
  __syncthreads();
  // group end = next group's start - 1; rank = 0.5 * (start + end) + 1
  for (int t = threadIdx.x; t < n; t += kThreads) {
    const int s = gstart[t];
    int e = t;
    // the end of t's group: the last position sharing its start (groups are contiguous)
    // found by a forward walk only from the group start's owner position
    if (t == s) {
      while (e + 1 < n && gstart[e + 1] == s) ++e;
      const double r = 0.5 * double(s + e) + 1.0;
      for (int u = s; u <= e; ++u) rank[uint32_t(k[u] & 0xFFFFFFFFull)] = r;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) spearman_rows_kernel(const SpearmanArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  unsigned long long* k = reinterpret_cast<unsigned long long*>(sm);  // [kMaxN]
  double* ra = reinterpret_cast<double*>(k + kMaxN);                   // [kMaxN]
  double* rb = ra + kMaxN;                                             // [kMaxN]
  int* gstart = reinterpret_cast<int*>(rb + kMaxN);                    // [kMaxN]
  const int i = blockIdx.x % a.N;
  const int bh = blockIdx.x / a.N;
  const int b = bh / a.H, h = bh % a.H;
  const long long o = (long long)bh * a.N + i;
  if (i == 0) {  // the reference starts at i = 1
    if (threadIdx.x == 0) a.defined[o] = 0, a.row_val[o] = 0.0;
    return;
  }
  const int n = i + 1;
  const float* pa = a.proxy + ((long long)(b * (a.H / a.c_h) + h / a.c_h) * a.N + i) * a.N;
  const float* pb = a.ref + o * a.N;
  average_ranks(pa, n, k, gstart, ra);
  average_ranks(pb, n, k, gstart, rb);
  if (threadIdx.x == 0) {
    const double mean = (double(n) + 1.0) / 2.0;
    double va = 0.0, vb = 0.0, cov = 0.0;
    for (int j = 0; j < n; ++j) {
      const double da = __dadd_rn(ra[j], -mean), db = __dadd_rn(rb[j], -mean);
      va = __dadd_rn(va, __dmul_rn(da, da));
      vb = __dadd_rn(vb, __dmul_rn(db, db));
      cov = __dadd_rn(cov, __dmul_rn(da, db));
    }
    const bool def = !(va == 0.0 || vb == 0.0);
    a.defined[o] = def;
    a.row_val[o] = def ? cov / sqrt(__dmul_rn(va, vb)) : 0.0;
  }
}

// ---------------------------------------------------------------- planted_recall
// metrics.cpp:178-199: per (b, h, i) with a non-empty planted list, the fraction of
// planted blocks the mask selected; planted = int32 [B][H][N][m], -1 = unused slot.
__global__ void planted_rows_kernel(int B, int H, int N, int W, int planes, int heads_per_plane, int m,
                                    const uint32_t* __restrict__ mask, const int32_t* __restrict__ planted,
                                    double* __restrict__ row_val, uint8_t* __restrict__ defined) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)B * H * N) return;
  const int i = int(r % N);
  const long long bh = r / N;
  const int b = int(bh / H), h = int(bh % H);
  const uint32_t* mrow = mask + ((long long)(b * planes + h / heads_per_plane) * N + i) * W;
  const int32_t* want = planted + r * m;
  int w = 0, hit = 0;
  for (int t = 0; t < m; ++t) {
    const int j = want[t];
    if (j < 0 || j >= N) continue;
    ++w;
    hit += (mrow[j >> 5] >> (j & 31)) & 1u;
  }
  defined[r] = w > 0;
  row_val[r] = w > 0 ? double(hit) / double(w) : 0.0;
}

// kMaskedScore (types.hpp:32) above the diagonal of [planes][N][N] block scores
__global__ void fill_upper_kernel(float* s, int N) {
  const int i = blockIdx.x % N;
  float* row = s + (long long)blockIdx.x * N;
  for (int j = i + 1 + threadIdx.x; j < N; j += blockDim.x) row[j] = -FLT_MAX;
}

constexpr size_t kSpearmanSmem = size_t(kMaxN) * (8 + 8 + 8 + 4);

}  // namespace

us_status launch_fill_upper(float* scores, long long planes, int N, cudaStream_t st) {
  fill_upper_kernel<<<unsigned(planes * N), 128, 0, st>>>(scores, N);
  US_LAUNCH_CHECK("fill_upper_kernel");
  return US_OK;
}

us_status launch_planted_recall(int B, int H, int N, int W, int planes, int heads_per_plane, int m,
                                const uint32_t* mask, const int32_t* planted, double* rows_ws, uint8_t* defined,
                                double* out, long long* n_def, cudaStream_t st) {
  const long long rows = (long long)B * H * N;
  planted_rows_kernel<<<unsigned((rows + 255) / 256), 256, 0, st>>>(B, H, N, W, planes, heads_per_plane, m, mask,
                                                                    planted, rows_ws, defined);
  US_LAUNCH_CHECK("planted_rows_kernel");
  ordered_mean_kernel<<<1, 32, 0, st>>>(rows, rows_ws, defined, out, n_def);
  US_LAUNCH_CHECK("ordered_mean_kernel");
  return US_OK;
}

us_status launch_output_fidelity(long long rows, int d, const uint16_t* test, const uint16_t* ref, double* rows_ws,
                                 double* out3, cudaStream_t st) {
  const unsigned grid = unsigned((rows + 127) / 128);
  fidelity_rows_kernel<<<grid, 128, 0, st>>>(rows, d, test, ref, rows_ws, rows_ws + rows, rows_ws + 2 * rows);
  US_LAUNCH_CHECK("fidelity_rows_kernel");
  fidelity_final_kernel<<<1, 32, 0, st>>>(rows, d, rows_ws, rows_ws + rows, rows_ws + 2 * rows, out3);
  US_LAUNCH_CHECK("fidelity_final_kernel");
  return US_OK;
}

us_status launch_block_recall(int B, int H, int N, int W, int planes, int heads_per_plane, int k,
                              const uint32_t* mask, const float* ref, double* rows_ws, double* out,
                              cudaStream_t st) {
  RecallArgs a{B, H, N, W, planes, heads_per_plane, k, mask, ref, rows_ws};
  recall_rows_kernel<<<unsigned((long long)B * H * N), kThreads, 0, st>>>(a);
  US_LAUNCH_CHECK("recall_rows_kernel");
  ordered_mean_kernel<<<1, 32, 0, st>>>((long long)B * H * N, rows_ws, nullptr, out, nullptr);
  US_LAUNCH_CHECK("ordered_mean_kernel");
  return US_OK;
}

us_status launch_row_spearman(int B, int H, int N, int c_h, const float* proxy, const float* ref, double* rows_ws,
                              uint8_t* defined, double* out, long long* n_def, cudaStream_t st) {
  static std::atomic<uint64_t> attr_done{0};
  if (us_status s = ensure_smem_attr(spearman_rows_kernel, int(kSpearmanSmem), attr_done,
                                     "spearman_rows_kernel smem attribute");
      s != US_OK)
    return s;
  SpearmanArgs a{B, H, N, c_h, proxy, ref, rows_ws, defined};
  spearman_rows_kernel<<<unsigned((long long)B * H * N), kThreads, kSpearmanSmem, st>>>(a);
  US_LAUNCH_CHECK("spearman_rows_kernel");
  ordered_mean_kernel<<<1, 32, 0, st>>>((long long)B * H * N, rows_ws, defined, out, n_def);
  US_LAUNCH_CHECK("ordered_mean_kernel");
  return US_OK;
}

}  // namespace us
