// compress.cu — multi-granularity compression.
//
// Reference: pool_sequence Mean (compression.hpp:26-28) then pool_heads
// (compression.hpp:61-76), driven by compress (compression.cpp:5-25).
//
// Bit-exactness: each window is summed in fp64 in row order, divided by c in
// fp64 and rounded once to f32; head groups are then summed in fp64 in member
// order, divided by c_h and rounded again — the reference's two roundings. For
// bf16 (and f32) inputs the fp64 window sum is exact, so the result does not
// depend on summation order and matches the reference/oracle bit for bit.
//
// Memory plan: one thread owns 8 consecutive d-elements of one output row and
// streams c rows of 16 B (8 x bf16) each: a warp covers 2 rows x 256 B, fully
// coalesced 128-bit loads, several loads in flight per thread. HBM-bound:
// bytes = planes_in * L * d * 2 (read) + planes_out * (L/c) * d * 4 (write).
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

__device__ __forceinline__ void bf16x8_to_f64_add(const uint4 v, double (&acc)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    acc[2 * t] += double(__uint_as_float(w[t] << 16));
    acc[2 * t + 1] += double(__uint_as_float(w[t] & 0xFFFF0000u));
  }
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 8 consecutive input elements of row `row` (in units of rows of d elements) as f32:
// bf16 storage (one 16-byte load) or f32 storage (two), both exact.
template <bool F32>
__device__ __forceinline__ void load8(const void* base, long long elem, float (&x)[8]) {
  if (F32) {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const float*>(base) + elem);
    const uint4 a = ld_stream(p), b = ld_stream(p + 1);
    x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y); x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
    x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y); x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
  } else {
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + elem));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[2 * q] = __uint_as_float(w[q] << 16);
      x[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  }
}

// inv: exact reciprocal when the divisor is a power of two (then x*inv == x/div
// bit for bit), else 0 and a true fp64 division is used.
__device__ __forceinline__ double divide(double x, double div, double inv) {
  return inv != 0.0 ? x * inv : x / div;
}

// SplitMix64 counter RNG and seed chaining of the reference (rng.hpp:11-67).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ uint64_t chain_seed(uint64_t s, uint64_t tag) { return mix64(s + kGamma + tag); }

// Sum over the `width` consecutive lanes that share one output row, reduced to
// the group's first lane in a fixed tree and broadcast, so every lane of the
// group holds the identical value.
__device__ __forceinline__ double group_sum(double v, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, width);
  return __shfl_sync(0xffffffffu, v, 0, width);
}

// STRAT: the pooling strategy, compile-time so the mean kernel (the default path)
// carries no registers for the max / stochastic code.
// F32: f32 input storage (the reference's own HeadStack<float>, C1): every strategy
// sums in fp64 in row order like the oracle; the bf16 fp32-exact fast path is skipped.
template <int STRAT, bool F32>
#ifndef US_COMPRESS_MINB  // resident 256-thread CTAs asked of ptxas for the mean kernel
#define US_COMPRESS_MINB 3
#endif
__global__ void __launch_bounds__(256, STRAT == US_POOL_MEAN ? US_COMPRESS_MINB : 1) compress_kernel(CompressArgs a, double inv_c, double inv_m) {
  const int chunks = a.d / 8;
  const int Lc = a.L / a.c;
  const long long total = (long long)a.B * a.planes * Lc * chunks;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = tid < total;
  // inactive lanes mirror the last row: the stochastic path shuffles across the
  // lanes of a row group, so every lane of a warp runs it
  const long long tid_eff = active ? tid : total - chunks + tid % chunks;
  float res[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int plane_id = 0;
  {
    const int ch = int(tid_eff % chunks);
    long long r = tid_eff / chunks;
    const int t = int(r % Lc);
    r /= Lc;
    const int p = int(r % a.planes);
    const int b = int(r / a.planes);
    plane_id = b * a.planes + p;
    double hacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int g = 0; g < a.members; ++g) {
      const int h = p * a.members + g;  // head index in the reference's (expanded) numbering
      const int hs = h / a.div;
      const long long elem0 = (((long long)b * a.H_src + hs) * a.L + (long long)t * a.c) * a.d + ch * 8;
      const uint4* src = reinterpret_cast<const uint4*>(a.src + (F32 ? 0 : elem0));
      const int stride = a.d / 8;  // uint4 per row (bf16)
      float val[8];
      bool done = false;
      if (!F32 && STRAT == US_POOL_MEAN && a.c > 1 && inv_c != 0.0) {
        // fp32 fast path: the running sum (from +0, row order, round-to-nearest) is
        // kept only if every addition was exact (round-down == round-up), so it
        // equals the fp64 sum; times the exact 1/c it rounds like the fp64 path
        // (denormals included). Any inexact step (wide exponent spread, overflow,
        // NaN) falls through to the fp64 path below.
        float sacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bool exact = true;
        for (int rr = 0; rr < a.c; rr += 8) {
          uint4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = u < a.c - rr ? ld_stream(src + (rr + u) * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (u >= a.c - rr) break;
            const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float x0 = __uint_as_float(w[q] << 16), x1 = __uint_as_float(w[q] & 0xFFFF0000u);
              exact &= __fadd_rd(sacc[2 * q], x0) == __fadd_ru(sacc[2 * q], x0);
              exact &= __fadd_rd(sacc[2 * q + 1], x1) == __fadd_ru(sacc[2 * q + 1], x1);
              sacc[2 * q] = __fadd_rn(sacc[2 * q], x0);
              sacc[2 * q + 1] = __fadd_rn(sacc[2 * q + 1], x1);
            }
          }
        }
        if (exact) {
          const float inv_cf = float(inv_c);
#pragma unroll
          for (int e = 0; e < 8; ++e) val[e] = __fmul_rn(sacc[e], inv_cf);
          done = true;
        }
      }
      if (done) {
      } else if (STRAT == US_POOL_MEAN || a.c == 1) {
        // (c == 1 returns the window row unchanged for every strategy, compression.hpp:20)
        // (the fp64 path: c == 1, non-power-of-two c, or a window the fp32 path
        // could not sum exactly — rare, so one row in flight keeps registers low)
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (F32) {
          for (int rr = 0; rr < a.c; ++rr) {
            float x[8];
            load8<true>(a.src, elem0 + (long long)rr * a.d, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += double(x[e]);
          }
        } else {
          for (int rr = 0; rr < a.c; ++rr) bf16x8_to_f64_add(ld_stream(src + rr * stride), acc);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) val[e] = __double2float_rn(divide(acc[e], double(a.c), inv_c));
      } else if (STRAT == US_POOL_MAX) {
        // column max over the window (compression.hpp:30-32); exact
#pragma unroll
        for (int e = 0; e < 8; ++e) val[e] = -INFINITY;
        for (int rr = 0; rr < a.c; ++rr) {
          float x[8];
          load8<F32>(a.src, elem0 + (long long)rr * a.d, x);
#pragma unroll
          for (int e = 0; e < 8; ++e) val[e] = fmaxf(val[e], x[e]);
        }
      } else {
        // stochastic (compression.hpp:33-53): pick window row r with probability
        // |row r| / sum of row norms, drawn from CounterRng(chain(chain(seed, role, h), t)).
        // Row norms: fp64 sums of squares (exact for bf16 inputs), sqrt, summed in row order.
        uint64_t state = chain_seed(chain_seed(chain_seed(a.seed, uint64_t(a.role)), uint64_t(a.head0 + h)), uint64_t(t));
        auto row_norm = [&](int rr) {
          float x[8];
          load8<F32>(a.src, elem0 + (long long)rr * a.d, x);
          double s2 = 0.0;
#pragma unroll
          for (int e = 0; e < 8; ++e) s2 += double(x[e]) * double(x[e]);
          return sqrt(group_sum(s2, chunks));
        };
        double tot = 0.0;
        for (int rr = 0; rr < a.c; ++rr) tot += row_norm(rr);
        int pick = a.c - 1;
        state += kGamma;
        const uint64_t draw = mix64(state);
        if (tot > 0.0) {
          const double u = double(draw >> 11) * 0x1.0p-53 * tot;
          double cum = 0.0;
          bool found = false;
          for (int rr = 0; rr < a.c; ++rr) {  // fixed trip count: shuffles stay warp-uniform
            cum += row_norm(rr);
            if (!found && u < cum) {
              pick = rr;
              found = true;
            }
          }
        } else {
          pick = int(draw % uint64_t(a.c));
        }
        load8<F32>(a.src, elem0 + (long long)pick * a.d, val);
      }
      if (a.members == 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) res[e] = val[e];
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) hacc[e] += double(val[e]);
      }
    }
    if (a.members > 1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) res[e] = __double2float_rn(divide(hacc[e], double(a.members), inv_m));
    }
    if (active && a.out) {
      float4* dst = reinterpret_cast<float4*>(a.out + (((long long)plane_id) * Lc + t) * a.d + ch * 8);
      dst[0] = make_float4(res[0], res[1], res[2], res[3]);
      dst[1] = make_float4(res[4], res[5], res[6], res[7]);
    }
    if (a.hi) {
      // fused split with a per-ROW power-of-two scale: the `chunks` lanes of the row
      // reduce its |max| (as f32 bits; NaN stays above everything), then each lane
      // writes x 2^e = hi + lo (fp16 pair, ~22 significant bits) for its 8 elements;
      // e makes the row's |max| * 2^e land in [2^14, 2^15) (the split_kernel rule per row)
      uint32_t mb = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float av = fabsf(res[e]);
        mb = max(mb, av != av ? 0x7FC00000u : __float_as_uint(av));
      }
      for (int o = chunks >> 1; o > 0; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o, chunks));
      const float amax = __uint_as_float(mb);
      int ex2 = 0;
      if (amax > 0.f && amax < INFINITY) {
        int ex;
        frexpf(amax, &ex);
        ex2 = 15 - ex;
      }
      __half h[8], l[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float x = ldexpf(res[e], ex2);
        h[e] = __float2half_rn(x);
        l[e] = __float2half_rn(x - __half2float(h[e]));
      }
      if (active) {
        const long long o = (((long long)plane_id) * Lc + t) * a.d + ch * 8;
        uint4 hv, lv;
        hv.x = uint32_t(__half_as_ushort(h[0])) | (uint32_t(__half_as_ushort(h[1])) << 16);
        hv.y = uint32_t(__half_as_ushort(h[2])) | (uint32_t(__half_as_ushort(h[3])) << 16);
        hv.z = uint32_t(__half_as_ushort(h[4])) | (uint32_t(__half_as_ushort(h[5])) << 16);
        hv.w = uint32_t(__half_as_ushort(h[6])) | (uint32_t(__half_as_ushort(h[7])) << 16);
        lv.x = uint32_t(__half_as_ushort(l[0])) | (uint32_t(__half_as_ushort(l[1])) << 16);
        lv.y = uint32_t(__half_as_ushort(l[2])) | (uint32_t(__half_as_ushort(l[3])) << 16);
        lv.z = uint32_t(__half_as_ushort(l[4])) | (uint32_t(__half_as_ushort(l[5])) << 16);
        lv.w = uint32_t(__half_as_ushort(l[6])) | (uint32_t(__half_as_ushort(l[7])) << 16);
        *reinterpret_cast<uint4*>(a.hi + o) = hv;
        *reinterpret_cast<uint4*>(a.lo + o) = lv;
        if (ch == 0) a.row_exp[(long long)plane_id * Lc + t] = ex2;
      }
    }
  }
  if (a.absmax) {
    float m = 0.f;
    if (active) {
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(res[e]));
      // NaN sorts above every finite value as unsigned bits; keep it visible.
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (res[e] != res[e]) m = __uint_as_float(0x7FC00000u);
    }
    const unsigned full = __activemask();
    const int leader_plane = __shfl_sync(full, plane_id, 0);
    const bool uniform = __all_sync(full, !active || plane_id == leader_plane);
    uint32_t bits = __float_as_uint(m);
    if (uniform) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bits = max(bits, __shfl_xor_sync(full, bits, o));
      if ((threadIdx.x & 31) == 0 && bits) atomicMax(a.absmax + leader_plane, bits);
    } else if (active && bits) {
      atomicMax(a.absmax + plane_id, bits);
    }
  }
}

__global__ void __launch_bounds__(256) split_kernel(SplitArgs a) {
  const long long per_plane = (long long)a.rows * a.d;
  const long long n4 = (long long)a.planes_total * per_plane / 4;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n4;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e0 = q * 4;
    const int plane = int(e0 / per_plane);
    const float amax = __uint_as_float(a.absmax[plane]);
    // e: amax * 2^e in [2^14, 2^15) keeps hi within fp16 range with headroom.
    int e = 0;
    if (amax > 0.f && amax < INFINITY) {
      int ex;
      frexpf(amax, &ex);  // amax = f * 2^ex, f in [0.5, 1)
      e = 15 - ex;
    }
    if (e0 % per_plane == 0) a.exp_out[plane] = e;
    const float4 v = reinterpret_cast<const float4*>(a.in)[q];
    const float x[4] = {ldexpf(v.x, e), ldexpf(v.y, e), ldexpf(v.z, e), ldexpf(v.w, e)};
    __half h[4], l[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      h[t] = __float2half_rn(x[t]);
      l[t] = __float2half_rn(x[t] - __half2float(h[t]));
    }
    reinterpret_cast<uint2*>(a.hi)[q] =
        make_uint2(uint32_t(__half_as_ushort(h[0])) | (uint32_t(__half_as_ushort(h[1])) << 16),
                   uint32_t(__half_as_ushort(h[2])) | (uint32_t(__half_as_ushort(h[3])) << 16));
    reinterpret_cast<uint2*>(a.lo)[q] =
        make_uint2(uint32_t(__half_as_ushort(l[0])) | (uint32_t(__half_as_ushort(l[1])) << 16),
                   uint32_t(__half_as_ushort(l[2])) | (uint32_t(__half_as_ushort(l[3])) << 16));
  }
}

__global__ void __launch_bounds__(256) f32_to_bf16_kernel(const float4* __restrict__ in, uint2* __restrict__ out,
                                                          long long n4) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x) {
    const float4 v = in[q];
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    out[q] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}

double exact_inverse(int c) { return (c > 0 && (c & (c - 1)) == 0) ? 1.0 / double(c) : 0.0; }

}  // namespace

us_status launch_compress(const CompressArgs& a, cudaStream_t st) {
  const long long total = (long long)a.B * a.planes * (a.L / a.c) * (a.d / 8);
  const int threads = 256;
  const long long blocks = (total + threads - 1) / threads;
  const double ic = exact_inverse(a.c), im = exact_inverse(a.members);
  const unsigned g = unsigned(blocks);
  if (a.src_f32) {
    if (a.strategy == US_POOL_MAX) compress_kernel<US_POOL_MAX, true><<<g, threads, 0, st>>>(a, ic, im);
    else if (a.strategy == US_POOL_STOCHASTIC) compress_kernel<US_POOL_STOCHASTIC, true><<<g, threads, 0, st>>>(a, ic, im);
    else compress_kernel<US_POOL_MEAN, true><<<g, threads, 0, st>>>(a, ic, im);
  } else {
    if (a.strategy == US_POOL_MAX) compress_kernel<US_POOL_MAX, false><<<g, threads, 0, st>>>(a, ic, im);
    else if (a.strategy == US_POOL_STOCHASTIC) compress_kernel<US_POOL_STOCHASTIC, false><<<g, threads, 0, st>>>(a, ic, im);
    else compress_kernel<US_POOL_MEAN, false><<<g, threads, 0, st>>>(a, ic, im);
  }
  US_LAUNCH_CHECK("compress_kernel");
  return US_OK;
}

us_status launch_f32_to_bf16(const float* in, void* out, long long n, cudaStream_t st) {
  if (n % 4) {
    set_error("f32 -> bf16 conversion: element count must be a multiple of 4");
    return US_ERR_UNSUPPORTED;
  }
  const long long n4 = n / 4;
  long long blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (n4 > 0)
    f32_to_bf16_kernel<<<unsigned(blocks), 256, 0, st>>>(reinterpret_cast<const float4*>(in),
                                                          static_cast<uint2*>(out), n4);
  US_LAUNCH_CHECK("f32_to_bf16_kernel");
  return US_OK;
}

us_status launch_split(const SplitArgs& a, cudaStream_t st) {
  const long long n4 = (long long)a.planes_total * a.rows * a.d / 4;
  const int threads = 256;
  long long blocks = (n4 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  split_kernel<<<unsigned(blocks), threads, 0, st>>>(a);
  US_LAUNCH_CHECK("split_kernel");
  return US_OK;
}

}  // namespace us
