// host_util.hpp — host-side helpers shared by the C-ABI translation units:
// thread-local error text, CUDA error mapping, TMA tensor-map encoding through
// the driver entry point (no link-time dependency on libcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/us_api.h"

namespace us {

void set_error(const std::string& msg);
int& launch_counter();

inline us_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return US_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return US_ERR_CUDA;
}

#define US_CUDA_TRY(expr, what)                                   \
  do {                                                            \
    us_status _s = ::us::cuda_status((expr), what);               \
    if (_s != US_OK) return _s;                                   \
  } while (0)

#define US_LAUNCH_CHECK(what)                                     \
  do {                                                            \
    ++::us::launch_counter();                                     \
    us_status _s = ::us::cuda_status(cudaGetLastError(), what);   \
    if (_s != US_OK) return _s;                                   \
  } while (0)

// Dynamic shared memory above 48 KB is a per-DEVICE function attribute: set it once
// per device ordinal (bit d of `done`; devices >= 64 set it on every launch). Two
// threads racing on the same device both set the same value, which is harmless.
template <typename Kernel>
inline us_status ensure_smem_attr(Kernel* fn, int bytes, std::atomic<uint64_t>& done, const char* what) {
  int dev = 0;
  US_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return US_OK;
  US_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
  done.fetch_or(bit, std::memory_order_release);
  return US_OK;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2D row-major tensor [rows][cols] of 16-bit elements, box [box_rows][box_cols],
// SWIZZLE_128B (box_cols * 2 must be 128 bytes).
inline us_status make_tmap_2d_16b(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                                  uint32_t box_rows, uint32_t box_cols, bool bf16) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return US_ERR_CUDA;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return US_ERR_CUDA;
  }
  return US_OK;
}

// K / V rows [rows][D] bf16 as a 3-D map (64 elements, rows, D/64 chunks) with a
// box of (64, box_rows, D/64): ONE TMA brings a box_rows x D tile into smem as
// [chunk][row][128 B] (SWIZZLE_128B per 128-byte line), the layout of two
// separate 2-D chunk loads.
inline us_status make_tmap_rows_chunked(CUtensorMap* m, const void* base, uint64_t rows, uint32_t D,
                                        uint32_t box_rows) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return US_ERR_CUDA;
  }
  cuuint64_t dims[3] = {64, rows, D / 64};
  cuuint64_t strides[2] = {uint64_t(D) * 2, 128};
  cuuint32_t box[3] = {64, box_rows, D / 64};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3-D rows x chunks) failed (" + std::to_string(int(r)) + ")");
    return US_ERR_CUDA;
  }
  return US_OK;
}

}  // namespace us
