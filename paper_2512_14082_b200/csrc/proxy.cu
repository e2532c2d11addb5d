// proxy.cu — compressed proxy attention on tcgen05.
//
// Reference: compressed_attention (proxy.cpp:10-46) and block_aggregate
// (proxy.cpp:48-72): logits = Qc.Kc^T / sqrt(d) in fp64, softmax per composite
// row over all composite keys (post-softmax, the default) or over the live
// prefix (pre-softmax, live iff (t'+1)c_q - 1 >= s' c_k), then per
// (query block i, key block j <= i) region sums.
//
// Precision ("fp16x3"): Qc/Kc are f32. The split kernel stores x * 2^e as
// hi = fp16(x 2^e), lo = fp16(x 2^e - hi) (~22 significant bits). Each logit
// tile is accumulated by three tcgen05 MMAs into one fp32 TMEM accumulator:
// hi.hi + hi.lo + lo.hi (the dropped lo.lo term is < 2^-22 relative). This is
// fp32-class accuracy at bf16 tensor-core rate — plain bf16/tf32 composite
// tokens flip mask bits vs the fp64 reference.
//
// Work split (the row LSE needs every key before any score can be formed):
//   pass 1: CTA = 128 composite query rows; streams all key tiles (post) or the
//           live ones (pre); online max/sum in log2 units -> lse2[row].
//   pass 2: same CTA tiling over causal key tiles only; p = 2^(x - lse2),
//           region sums over rk keys (thread-local) and rq rows (warp shuffles,
//           fixed tree) -> scores[i][j], j <= i.
//
// Roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (+TMEM owner),
// warps 2..5 epilogue; epilogue warp w owns TMEM lanes 32*(w%4).. (row = lane).
// Pipelines: K tiles double-buffered in smem (k_full/k_empty), S accumulators
// double-buffered in TMEM (s_full/s_empty) so tile t+1's MMAs overlap tile t's
// exp work.
#include "host_util.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace us {
namespace {

constexpr int kRows = 128;  // composite query rows per CTA (UMMA M)
constexpr int kKeys = 128;  // composite keys per tile (UMMA N)
constexpr int kStages = 2;

template <int D>
struct ProxySmem {
  static constexpr int kChunks = D / 64;                 // 128-byte swizzle atoms along d
  static constexpr int kQBytes = kRows * D * 2;          // one of hi/lo
  static constexpr int kKBytes = kKeys * D * 2;          // one of hi/lo
  static constexpr int kQOff = 0;                        // Qh, Ql
  static constexpr int kKOff = 2 * kQBytes;              // stage s: Kh, Kl
  static constexpr int kBytes = kKOff + kStages * 2 * kKBytes;
};

__device__ __forceinline__ int live_keys(int t, int c_q, int c_k, int Lk, int mode) {
  if (mode == US_POST_SOFTMAX_BLOCK_CAUSAL) return Lk;
  const long long last_q = (long long)(t + 1) * c_q - 1;
  const long long live = last_q / c_k + 1;
  return live < Lk ? int(live) : Lk;
}

template <int D, int PASS>
__global__ void __launch_bounds__(192, 1)
    proxy_kernel(const __grid_constant__ CUtensorMap tmQh, const __grid_constant__ CUtensorMap tmQl,
                 const __grid_constant__ CUtensorMap tmKh, const __grid_constant__ CUtensorMap tmKl,
                 const ProxyArgs a) {
  using L = ProxySmem<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_q, bar_kfull[kStages], bar_kempty[kStages], bar_sfull[2], bar_sempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float red[kRows][33];  // pass 2: per-row key-group partials of one segment

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rt = gridDim.x - 1 - blockIdx.x;  // heavy (late) row tiles first
  const int hc = blockIdx.y, b = blockIdx.z;
  const int r0 = rt * kRows;
  const int plane = b * a.Hc + hc;
  const int kvp = (hc * a.kv_mul) / a.kv_div;
  const int kplane = b * a.kv_planes + kvp;

  // key-tile range
  const int r_last = min(r0 + kRows, a.Lq) - 1;
  int nkeys;
  if (PASS == 1) {
    nkeys = live_keys(r_last, a.c_q, a.c_k, a.Lk, a.causal_mode);
  } else {
    const int i_max = r_last / a.rq;
    nkeys = min(a.Lk, (i_max + 1) * a.rk);
  }
  const int n_tiles = (nkeys + kKeys - 1) / kKeys;

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar_kfull[s], 1);
      mbar_init(&bar_kempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sempty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      tma_prefetch_desc(&tmQh);
      tma_prefetch_desc(&tmKh);
      const int qrow = plane * a.Lq + r0;
      mbar_arrive_expect_tx(&bar_q, 2 * L::kQBytes);
      for (int kc = 0; kc < L::kChunks; ++kc) {
        tma_load_2d(smem + L::kQOff + kc * kRows * 128, &tmQh, &bar_q, kc * 64, qrow);
        tma_load_2d(smem + L::kQOff + L::kQBytes + kc * kRows * 128, &tmQl, &bar_q, kc * 64, qrow);
      }
      const uint64_t pol = policy_evict_last();  // K tiles are re-read by every row tile
      for (int t = 0; t < n_tiles; ++t) {
        const int s = t % kStages;
        if (t >= kStages) mbar_wait(&bar_kempty[s], ((t / kStages) + 1) & 1);
        uint8_t* kh = smem + L::kKOff + s * 2 * L::kKBytes;
        uint8_t* kl = kh + L::kKBytes;
        mbar_arrive_expect_tx(&bar_kfull[s], 2 * L::kKBytes);
        const int krow = kplane * a.Lk + t * kKeys;
        for (int kc = 0; kc < L::kChunks; ++kc) {
          tma_load_2d_hint(kh + kc * kKeys * 128, &tmKh, &bar_kfull[s], kc * 64, krow, pol);
          tma_load_2d_hint(kl + kc * kKeys * 128, &tmKl, &bar_kfull[s], kc * 64, krow, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_f16(kRows, kKeys, /*f16*/ 0, false, false);
    mbar_wait(&bar_q, 0);
    tc_fence_after();
    for (int t = 0; t < n_tiles; ++t) {
      const int s = t % kStages, buf = t & 1;
      mbar_wait(&bar_kfull[s], (t / kStages) & 1);
      if (t >= 2) mbar_wait(&bar_sempty[buf], ((t - 2) / 2) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t qh = smem_u32(smem + L::kQOff), ql = qh + L::kQBytes;
        const uint32_t kh = smem_u32(smem + L::kKOff + s * 2 * L::kKBytes), kl = kh + L::kKBytes;
        const uint32_t d_tmem = tmem + buf * kKeys;
#pragma unroll
        for (int kc = 0; kc < L::kChunks; ++kc) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t qo = kc * kRows * 128 + ks * 32, ko = kc * kKeys * 128 + ks * 32;
            const uint64_t aqh = sdesc_sw128(qh + qo, 16, 1024), aql = sdesc_sw128(ql + qo, 16, 1024);
            const uint64_t bkh = sdesc_sw128(kh + ko, 16, 1024), bkl = sdesc_sw128(kl + ko, 16, 1024);
            umma_f16_ss(d_tmem, aqh, bkl, idesc, (kc | ks) != 0);
            umma_f16_ss(d_tmem, aql, bkh, idesc, 1);
            umma_f16_ss(d_tmem, aqh, bkh, idesc, 1);
          }
        }
        umma_commit(&bar_kempty[s]);
        umma_commit(&bar_sfull[buf]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter
    const int row = q * 32 + lane;
    const int t_row = r0 + row;
    const bool row_ok = t_row < a.Lq;
    const int live = row_ok ? live_keys(t_row, a.c_q, a.c_k, a.Lk, a.causal_mode) : 0;
    const float k2 = ldexpf(a.scale_log2, -(a.exp_q[plane] + a.exp_k[kplane]));
    const uint32_t lane_addr = tmem + (uint32_t(q * 32) << 16);
    float m = -INFINITY, l = 0.f;
    const float lse2 = (PASS == 2 && row_ok) ? a.lse2[(long long)plane * a.Lq + t_row] : 0.f;
    for (int t = 0; t < n_tiles; ++t) {
      const int buf = t & 1;
      mbar_wait(&bar_sfull[buf], (t / 2) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < kKeys / 32; ++ch) {
        uint32_t v[32];
        tmem_ld32(lane_addr + buf * kKeys + ch * 32, v);
        tmem_ld_wait();
        if (ch == kKeys / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_sempty[buf]);
        }
        const int key0 = t * kKeys + ch * 32;
        if (PASS == 1) {
          float x[32];
          float cm = -INFINITY;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            x[c] = (key0 + c < live) ? __uint_as_float(v[c]) * k2 : -INFINITY;
            cm = fmaxf(cm, x[c]);
          }
          const float m_new = fmaxf(m, cm);
          if (m_new != -INFINITY) {
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < 32; ++c) sum += ex2_approx(x[c] - m_new);
            l = l * ex2_approx(m - m_new) + sum;
            m = m_new;
          }
        } else {
          float v32[32];
#pragma unroll
          for (int c = 0; c < 32; ++c)
            v32[c] = (key0 + c < live) ? ex2_approx(fmaf(__uint_as_float(v[c]), k2, -lse2)) : 0.f;
          // pairwise tree inside groups of min(rk, 32) keys (register indices are
          // compile-time; the runtime rk only predicates whole levels)
#pragma unroll
          for (int w = 1; w < 32; w <<= 1) {
            if (w < a.rk) {
#pragma unroll
              for (int c = 0; c < 32; c += 2 * w) v32[c] += v32[c + w];
            }
          }
          // stage this row's key-group partials of the current segment in smem
          const int cps = min(4, a.rk);            // chunks per segment
          const int gseg = (32 * cps) / a.rk;      // key groups per segment (<= 32)
          const int cseg = ch % cps;               // chunk index inside the segment
          if (a.rk <= 32) {
            const int ng = 32 / a.rk;
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if ((c & (a.rk - 1)) == 0) red[row][cseg * ng + c / a.rk] = v32[c];
          } else {
            const int gi = (cseg * 32) / a.rk;     // group inside the segment
            if ((cseg * 32) % a.rk == 0) red[row][gi] = v32[0];
            else red[row][gi] += v32[0];
          }
          if (cseg == cps - 1) {
            // cross-row sums over the rq rows of each query block, fixed order,
            // consecutive threads -> consecutive key blocks (coalesced stores)
            named_bar_sync(1, 128);
            const int qb_tile = kRows / a.rq;
            const int nout = qb_tile * gseg;
            const int j0 = (t * kKeys + (ch - cseg) * 32) / a.rk;
            for (int o = row; o < nout; o += 128) {
              const int qb = o / gseg, gg = o % gseg;
              float sum = 0.f;
              for (int r = 0; r < a.rq; ++r) sum += red[qb * a.rq + r][gg];
              const int i = (r0 / a.rq) + qb;
              const int j = j0 + gg;
              if (qb * a.rq + r0 < a.Lq && j <= i)
                a.scores[((long long)plane * a.N + i) * a.N + j] = sum;
            }
            named_bar_sync(1, 128);
          }
        }
      }
    }
    if (PASS == 1 && row_ok) a.lse2[(long long)plane * a.Lq + t_row] = m + __log2f(l);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

template <int D, int PASS>
us_status launch_proxy_t(const ProxyArgs& a, const CUtensorMap& tmQh, const CUtensorMap& tmQl,
                         const CUtensorMap& tmKh, const CUtensorMap& tmKl, cudaStream_t st) {
  const int smem = ProxySmem<D>::kBytes + 1024;
  auto kern = proxy_kernel<D, PASS>;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    US_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                "proxy_kernel smem attribute");
    attr_set = true;
  }
  dim3 grid((a.Lq + kRows - 1) / kRows, a.Hc, a.B);
  kern<<<grid, 192, smem, st>>>(tmQh, tmQl, tmKh, tmKl, a);
  US_LAUNCH_CHECK("proxy_kernel");
  return US_OK;
}

}  // namespace

us_status launch_proxy(const ProxyArgs& a, const CUtensorMap& tmQh, const CUtensorMap& tmQl,
                       const CUtensorMap& tmKh, const CUtensorMap& tmKl, int pass,
                       cudaStream_t st) {
  if (a.D == 128)
    return pass == 1 ? launch_proxy_t<128, 1>(a, tmQh, tmQl, tmKh, tmKl, st)
                     : launch_proxy_t<128, 2>(a, tmQh, tmQl, tmKh, tmKl, st);
  if (a.D == 64)
    return pass == 1 ? launch_proxy_t<64, 1>(a, tmQh, tmQl, tmKh, tmKl, st)
                     : launch_proxy_t<64, 2>(a, tmQh, tmQl, tmKh, tmKl, st);
  set_error("proxy: d_k must be 64 or 128 on the GPU path");
  return US_ERR_UNSUPPORTED;
}

}  // namespace us
