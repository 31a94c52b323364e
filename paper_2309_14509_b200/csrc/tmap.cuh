// Host helper: TMA tensor maps over the reference's [s, b, h, hd] layout,
// encoded with cuTensorMapEncodeTiled fetched through the runtime's driver
// entry point (no link-time dependency on libcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ul {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline int get_encode_fn(EncodeTiledFn* out) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !ptr)
      return fail(UL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(e));
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  *out = fn;
  return UL_OK;
}

// 3-D bf16 map over a [rows, heads, hd] view of [s, b, h, hd] (heads = b*h):
// box = {64 hd elements (128 B, SWIZZLE_128B), 1 head, box_rows rows}.
inline int make_tmap_bhsd(CUtensorMap* m, const void* ptr, int64_t rows, int64_t heads, int64_t hd,
                          int box_rows) {
  EncodeTiledFn enc;
  UL_TRY(get_encode_fn(&enc));
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    return fail(UL_ERR_ARG, "attention operand not 16-byte aligned");
  cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)(hd * 2), (cuuint64_t)(heads * hd * 2)};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
#ifndef UL_TMAP_L2_PROMOTION
#define UL_TMAP_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, UL_TMAP_L2_PROMOTION,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return UL_OK;
}

}  // namespace ul

namespace ul {
// 2-D bf16 row-major matrix [rows, cols] (row stride = cols), SWIZZLE_128B
// boxes of 64 columns x box_rows rows; OOB rows/cols read as zero.
inline int make_tmap_2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn enc;
  UL_TRY(get_encode_fn(&enc));
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) != 0 || (cols * 2) % 16 != 0)
    return fail(UL_ERR_ARG, "GEMM operand not 16-byte aligned");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return UL_OK;
}
}  // namespace ul
